# shard-vs-single K1: ncu --set full of one K1 of each on the
# same 256^3 system, and the DRAM bytes of one whole P=1 shard solve (NVTX
# range dcg.loopback_solve -- also shows the NVTX ranges reach ncu)
mkdir -p gpurun_out
timeout 300 python scripts/shard_k1_probe.py
timeout 600 ncu --nvtx --nvtx-include "dcg.loopback_solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 44 --csv python scripts/shard_k1_probe.py > gpurun_out/shard_solve_dram.csv 2>&1; echo "ncu nvtx rc $?"; grep -c '"dram__bytes_read.sum"' gpurun_out/shard_solve_dram.csv
timeout 600 ncu --nvtx --nvtx-include "cg.solve/" --metrics gpu__time_duration.sum --clock-control none -c 50 --csv python scripts/shard_k1_probe.py > gpurun_out/nvtx_cg_solve.csv 2>&1; echo "ncu nvtx cg rc $?"; grep -c gpu__time_duration gpurun_out/nvtx_cg_solve.csv
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"DcgSpmvOp<.bool.0, .bool.0>, .int.7" -s 2 -c 1 -o gpurun_out/prof_shard_k1 -f python scripts/shard_k1_probe.py > gpurun_out/ncu_shard.log 2>&1; echo "ncu shard rc $?"; tail -2 gpurun_out/ncu_shard.log
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_spmv_tma<rvk::CgSpmvOp<.bool.0, .bool.0>, .int.7" -s 4 -c 1 -o gpurun_out/prof_single_k1 -f python scripts/shard_k1_probe.py > gpurun_out/ncu_single.log 2>&1; echo "ncu single rc $?"; tail -2 gpurun_out/ncu_single.log
