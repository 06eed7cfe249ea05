mkdir -p gpurun_out
for cfgname in 7pt256 27pt256 5pt1024; do
  for m in fused unfused; do
    timeout 300 python bench.py --solver tfqmr --config $cfgname --mode $m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tfq_${cfgname}_${m}.json 2> gpurun_out/tfq_${cfgname}_${m}.err; tail -1 gpurun_out/tfq_${cfgname}_${m}.err
  done
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cg.json 2> gpurun_out/cg.err; tail -1 gpurun_out/cg.err
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo parity rc $?; tail -2 gpurun_out/parity.log
