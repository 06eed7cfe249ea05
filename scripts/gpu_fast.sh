mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv or cg_vs or golden or headline or chunked" > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_fast.log
for c in 27pt256 9pt4096 7pt256; do for v in fast base fast base; do
if [ $v = base ]; then export RVK_LIB_PATH=$PWD/paper_2306_17801_b200/lib_ab/librvk.so; else unset RVK_LIB_PATH; fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > /dev/null 2> /tmp/e.err; echo "$c $v $(tail -1 /tmp/e.err)"
done; done
