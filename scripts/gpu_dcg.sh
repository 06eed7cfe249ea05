exec > gpurun_out/dcg.log 2>&1
RVK_OFF32=1 timeout 600 ncu --set full --clock-control none -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_off32 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc $?
