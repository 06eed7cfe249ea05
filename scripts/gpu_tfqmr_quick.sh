mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tfqmr.py -x -q > gpurun_out/pytest_tfqmr.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_tfqmr.log
for cfgname in 7pt256 27pt256 5pt1024; do
    timeout 300 python bench.py --solver tfqmr --config $cfgname --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tfq_${cfgname}.json 2> gpurun_out/tfq_${cfgname}.err; tail -1 gpurun_out/tfq_${cfgname}.err
done
A="--solver tfqmr --steps 1 --warmup 3 --no-cpu-baseline --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tfq_launches.csv python bench.py $A > gpurun_out/tfq_ll.log 2>&1; echo ll rc $?
