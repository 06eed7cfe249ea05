# plane-marching K1: parity tests, then 768^3 / 512^3 A/B (auto = march vs
# RVK_OPT_NO_MARCH = 2048) with ncu DRAM bytes of K1 launches
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_march.py tests/test_gpu_trace.py -q -x -p no:cacheprovider > gpurun_out/pytest_march.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_march.log
for c in 7pt768 7pt512; do for o in 0 2048; do
  echo "$c opts=$o $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c --opts $o 2>&1 >/dev/null | tail -1 | cut -c1-150)"
done; done
for o in 0 2048; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_spmv" -s 6 -c 2 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 7pt768 --opts $o > gpurun_out/march_ncu_$o.csv 2>/dev/null; echo "ncu $o rc $?"
done
