mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer_ipc.py -x -q -k bench > gpurun_out/pytest_bench2.log 2>&1; echo "rc $?"; tail -30 gpurun_out/pytest_bench2.log
