# Scratch A/B script for one-off GPU experiments (gpurun -- bash scripts/gpu_scratch.sh);
# its last contents are whatever experiment ran last -- not part of the round-end checks
# (those are scripts/gpu_final.sh and scripts/gpu_profiles.sh).
exec > gpurun_out/dcg.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_peer_ipc.py tests/test_gpu_parity.py -x -q -k "shard or peer or dcg or const or loopback" 2>&1 | tail -3
for i in 1 2; do timeout 300 python scripts/dcg_time.py 2>&1 | head -1; done
timeout 600 python scripts/peer_overhead.py 2>&1 | head -4
