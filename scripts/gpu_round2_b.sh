# full -m gpu suite, traced demo, latency sweep (auto = cluster / grid solve vs the fused graph),
# shard-vs-single K1 ncu capture
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -3; grep FAILED gpurun_out/pytest_gpu.log | head
timeout 300 python scripts/trace_demo.py gpurun_out/trace > gpurun_out/trace_demo.txt 2>&1; echo "trace rc $?"; head -30 gpurun_out/trace_demo.txt
for c in 5pt64 5pt128 5pt256 5pt512 5pt1024; do
  echo "$c auto  $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 20 --warmup 5 --config $c --mode auto 2>&1 >/dev/null | tail -1 | cut -c1-60)"
  echo "$c fused $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 20 --warmup 5 --config $c --mode fused 2>&1 >/dev/null | tail -1 | cut -c1-60)"
  echo "$c hostsync $(timeout 300 python bench.py --no-cpu-baseline --no-strong --steps 10 --warmup 3 --config $c --mode hostsync 2>&1 >/dev/null | tail -1 | cut -c1-60)"
done
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"DcgSpmvOp<0, 0>" -s 2 -c 1 -o gpurun_out/prof_shard_k1 -f python scripts/shard_k1_probe.py > /dev/null 2>&1; echo "ncu shard rc $?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_spmv_tma<CgSpmvOp<0, 0>" -s 4 -c 1 -o gpurun_out/prof_single_k1 -f python scripts/shard_k1_probe.py > /dev/null 2>&1; echo "ncu single rc $?"
