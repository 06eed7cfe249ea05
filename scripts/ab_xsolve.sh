exec > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or sharded or sanitizer" 2>&1 | tail -4
for c in 7pt256 27pt256 9pt4096; do
for g in solve 4; do
RVK_X_GROUP=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c 2>&1 >/dev/null | tail -1 | sed "s/^/$c g=$g /"
done; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 7pt768 2>&1 >gpurun_out/b768.json | tail -1
