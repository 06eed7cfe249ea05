# TFQMR parity on the GPU + C++ API + smoke
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tfqmr.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_tfqmr.log 2>&1; echo pytest rc $?; tail -25 gpurun_out/pytest_tfqmr.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -5 gpurun_out/smoke.log
