# Round profile capture: bench lines + ncu launch list + ncu --set full of the
# dominant kernels (summarised into profiles/ by scripts/make_profiles.py).
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc $?"; tail -1 gpurun_out/bench_default.err
for c in 27pt256 9pt4096 5pt1024 7pt768; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c $(tail -1 gpurun_out/bench_$c.err)"
done
for c in 7pt256 27pt256 9pt4096; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --operator stencil --config $c > gpurun_out/bench_mf_$c.json 2> gpurun_out/bench_mf_$c.err; echo "mf $c $(tail -1 gpurun_out/bench_mf_$c.err)"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --solver tfqmr > gpurun_out/bench_tfqmr.json 2> gpurun_out/bench_tfqmr.err; echo "tfqmr $(tail -1 gpurun_out/bench_tfqmr.err)"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 126 -c 84 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu launches rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu k1 rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_update -s 4 -c 1 -o gpurun_out/prof_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu k2 rc $?
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1_27pt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 27pt256 > /dev/null 2>&1; echo ncu k1 27pt rc $?
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1_9pt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 9pt4096 > /dev/null 2>&1; echo ncu k1 9pt rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1_768 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 7pt768 > /dev/null 2>&1; echo ncu k1 768 rc $?
timeout 600 ncu --nvtx --nvtx-include "dcg.loopback_solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 44 --csv python scripts/shard_k1_probe.py > gpurun_out/shard_solve_dram.csv 2>&1; echo ncu shard solve rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mf_tma -s 4 -c 1 -o gpurun_out/prof_mf -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --operator stencil > /dev/null 2>&1; echo ncu mf rc $?
timeout 600 ncu --set full --clock-control none -k regex:k_mf_tma -s 4 -c 1 -o gpurun_out/prof_mf_27pt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --operator stencil --config 27pt256 > /dev/null 2>&1; echo ncu mf 27pt rc $?
timeout 600 ncu --set full --clock-control none -k regex:k_cg_grid_l2 -s 3 -c 1 -o gpurun_out/prof_gridl2_768 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strong --config 5pt768 > /dev/null 2>&1; echo ncu grid_l2 rc $?
# summarise on the box (ncu CLI there), keep only the headline K1 report
PROFILES_OUT=gpurun_out/profiles_out python scripts/make_profiles.py r02 > gpurun_out/make_profiles.log 2>&1; echo "make_profiles rc $?"
for f in gpurun_out/prof_*.ncu-rep; do [ "$f" = gpurun_out/prof_k1.ncu-rep ] || rm -f "$f"; done
du -sh gpurun_out
