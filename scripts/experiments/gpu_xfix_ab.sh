# xfix own grid + k_dcg_update 3 blocks/SM A/B (abvar/new vs old)
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
for r in 1 2; do for v in new old; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  echo "$v $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 2>&1 >/dev/null | tail -1 | cut -c1-80)"
  echo "$v $(timeout 300 python scripts/shard_k1_probe.py 2>&1 | tail -1)"
done; done
cp abvar/new/librvk.so paper_2306_17801_b200/lib/librvk.so
timeout 600 ncu --nvtx --nvtx-include "dcg.loopback_solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 44 --csv python scripts/shard_k1_probe.py > gpurun_out/shard_solve_dram_new.csv 2>&1; echo "ncu rc $?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cg_xfix -c 2 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong > gpurun_out/xfix_single_new.csv 2>&1; echo "ncu2 rc $?"
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
