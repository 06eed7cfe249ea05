# 768^3 K1 L2-policy experiment: variants abvar/<v>/librvk.so (RVK_EXP_L2
# builds: 1 evict_last gathers + evict_first p/w stores, 2 = 1 + persisting
# L2 set-aside, 3 = evict_last gathers + set-aside, 4 = set-aside only).
mkdir -p gpurun_out
cp paper_2306_17801_b200/lib/librvk.so /tmp/librvk_main.so
timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_tfqmr.py tests/test_gpu_api.py -q -x -p no:cacheprovider > gpurun_out/pytest_trace.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_trace.log
for v in base l2v1 l2v2 l2v3 l2v4; do
  cp abvar/$v/librvk.so paper_2306_17801_b200/lib/librvk.so
  echo "$v $(timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --config 7pt768 2>&1 >/dev/null | grep -v '^\[exp\]' | tail -1 | cut -c1-150)"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_spmv_tma -s 6 -c 2 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 7pt768 > gpurun_out/l2exp_$v.csv 2>/dev/null; echo "ncu $v rc $?"
done
cp /tmp/librvk_main.so paper_2306_17801_b200/lib/librvk.so
