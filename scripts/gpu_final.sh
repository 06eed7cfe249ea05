# Round-end validation: GPU tests, smoke, default bench, reference arm.
mkdir -p gpurun_out
exec > gpurun_out/final.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc $?"; tail -1 gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc $?"; tail -c 600 gpurun_out/final_ref.json
