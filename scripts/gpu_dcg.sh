exec > gpurun_out/dcg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mf or stencil or virtual or tiny or matrix" 2>&1 | tail -3
for c in 7pt256 9pt4096 27pt256 5pt1024; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --operator stencil --config $c 2>&1 >/dev/null | tail -1 | sed "s/^/mf $c /"
done
