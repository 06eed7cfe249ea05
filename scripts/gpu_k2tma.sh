mkdir -p gpurun_out
RVK_K2_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cg_vs or golden or headline or while or host_many or misaligned" > gpurun_out/pytest_k2.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_k2.log
for c in 7pt256 27pt256; do for k in 1 0 1 0; do
RVK_K2_TMA=$k timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > /dev/null 2> /tmp/e.err; echo "$c k2tma=$k $(tail -1 /tmp/e.err)"
done; done
RVK_K2_TMA=1 timeout 600 ncu --set full --clock-control none -k regex:k_cg_update_tma -s 4 -c 1 -o gpurun_out/prof_k2tma -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc $?
