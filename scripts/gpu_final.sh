# Round-end check: full -m gpu suite, smoke(), default bench, reference arm,
# N=2 torchrun path with both ranks on one GPU (functional only)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep FAILED gpurun_out/pytest_gpu.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; cat gpurun_out/smoke.log | tail -4
bash scripts/gpu_bench_all.sh
