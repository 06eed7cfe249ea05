exec > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or stencil or mf" 2>&1 | tail -4
for c in 7pt256 27pt256 9pt4096; do
for g in solve 4; do
RVK_X_GROUP=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --operator stencil --config $c 2>&1 >/dev/null | tail -1 | sed "s/^/mf $c g=$g /"
done; done
