# Scratch A/B script for one-off GPU experiments (gpurun -- bash scripts/gpu_scratch.sh);
# its last contents are whatever experiment ran last -- not part of the round-end checks
# (those are scripts/gpu_final.sh and scripts/gpu_profiles.sh).
exec > gpurun_out/scratch.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for f in 1 0 1 0; do
RVK_FOLD_SETUP=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | tail -1 | cut -c1-90 | sed "s/^/fold=$f /"
done
RVK_FOLD_SETUP=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config 27pt256 2>&1 >/dev/null | tail -1 | cut -c1-90 | sed "s/^/27pt fold=1 /"
RVK_FOLD_SETUP=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config 27pt256 2>&1 >/dev/null | tail -1 | cut -c1-90 | sed "s/^/27pt fold=0 /"
