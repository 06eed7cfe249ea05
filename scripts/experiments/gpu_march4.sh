mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck python scripts/experiments/march_probe.py 512 512 8 > gpurun_out/march_sanitize.log 2>&1; echo "sanitizer rc $?"; grep -E "flags|hist rel|ERROR SUMMARY" gpurun_out/march_sanitize.log | head -4
timeout 1500 python -m pytest tests/test_gpu_march.py tests/test_gpu_grid_solve.py -q -p no:cacheprovider > gpurun_out/pytest_march.log 2>&1; echo "pytest rc $?"; tail -8 gpurun_out/pytest_march.log
for c in 7pt768 7pt512; do for o in 0 2048; do
  echo "$c opts=$o $(timeout 600 python bench.py --no-cpu-baseline --no-strong --steps 5 --warmup 3 --config $c --opts $o 2>&1 >/dev/null | tail -1 | cut -c1-150)"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_spmv" -s 6 -c 2 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 7pt768 > gpurun_out/march_ncu_0.csv 2>/dev/null; echo "ncu rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmv_march" -s 3 -c 1 -o gpurun_out/prof_march768 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 7pt768 > /dev/null 2>&1; echo "ncu full rc $?"
