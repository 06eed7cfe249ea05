mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_baseline_sizes.py -q -p no:cacheprovider -k "tfqmr" -s > gpurun_out/pytest_tfqmr_bs.log 2>&1; echo "pytest rc $?"; grep -E "TFQMR|passed|failed" gpurun_out/pytest_tfqmr_bs.log | tail -4
bash scripts/gpu_profiles.sh
