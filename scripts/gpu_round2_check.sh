# Round-2 first GPU pass: full -m gpu suite (with durations), then the bench pass.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt; free -g >> gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=30 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -45 gpurun_out/pytest_gpu.log
bash scripts/gpu_bench_all.sh
