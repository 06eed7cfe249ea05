mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "matrix_free or while" > gpurun_out/pytest_mf.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_mf.log
for c in 7pt256 27pt256 9pt4096 5pt1024; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --operator stencil --config $c > /dev/null 2> gpurun_out/mf_$c.err; echo "$c $(tail -1 gpurun_out/mf_$c.err)"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mf -s 4 -c 1 -o gpurun_out/prof_mf -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --operator stencil > /dev/null 2>&1; echo "ncu rc $?"
