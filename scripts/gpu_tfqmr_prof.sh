# launch list (per-kernel durations) of one fused TFQMR solve + full capture of KA / KM
mkdir -p gpurun_out
A="--solver tfqmr --steps 1 --warmup 3 --no-cpu-baseline --no-graph ${BENCH_ARGS}"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tfq_launches.csv python bench.py $A > gpurun_out/tfq_ll.log 2>&1; echo ll rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 200 -c 2 -o gpurun_out/prof_tfq_spmv -f python bench.py $A > gpurun_out/ncu_tfq1.log 2>&1; echo ncu1 rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tfq_merge -s 40 -c 1 -o gpurun_out/prof_tfq_merge -f python bench.py $A > gpurun_out/ncu_tfq2.log 2>&1; echo ncu2 rc $?
