exec > gpurun_out/dcg.log 2>&1
timeout 600 python scripts/peer_overhead.py 256x256x256
