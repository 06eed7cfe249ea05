# The driver's round-end commands, as a dry run + the ncu evidence for profiles/
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc $?"; cat gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"; cat gpurun_out/bench_ref.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo "torchrun rc $?"; tail -c 300 gpurun_out/bench_torchrun1.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 123 -c 82 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu launches rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu k1 rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_update -s 4 -c 1 -o gpurun_out/prof_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu k2 rc $?
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1_27pt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 27pt256 > /dev/null 2>&1; echo ncu k1 27pt rc $?
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_tma -s 4 -c 1 -o gpurun_out/prof_k1_9pt -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 9pt4096 > /dev/null 2>&1; echo ncu k1 9pt rc $?
