exec > gpurun_out/dcg.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python scripts/dcg_time.py 256x256x256 2>&1 | head -1
RVK_X_GROUP=2 timeout 300 python scripts/dcg_time.py 256x256x256 2>&1 | head -1
