exec > gpurun_out/dcg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tfqmr.py -x -q -k "irregular" 2>&1 | tail -8
