exec > gpurun_out/dcg.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cg_cluster -s 3 -c 1 -o gpurun_out/prof_cluster -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 5pt128 --mode auto > /dev/null 2>&1; echo rc $?
