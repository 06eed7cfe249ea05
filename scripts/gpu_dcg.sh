exec > gpurun_out/dcg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tfqmr.py -x -q 2>&1 | tail -3
for cd in 1 0; do
RVK_CONST_DIAG=$cd timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --solver tfqmr 2>&1 >/dev/null | tail -1 | sed "s/^/cd=$cd /"
RVK_CONST_DIAG=$cd timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --solver tfqmr --config 27pt256 2>&1 >/dev/null | tail -1 | sed "s/^/27pt cd=$cd /"
done
