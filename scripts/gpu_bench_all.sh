# Round bench pass: N=1 default line (headline + strong_768 anchor + CPU
# baseline), the reference arm, and the N=2 torchrun path with both ranks on
# one GPU (functional check of the sharded bench; timings meaningless).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "n1 rc $?"; tail -3 gpurun_out/bench_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"; tail -1 gpurun_out/bench_ref.err
RVK_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err; echo "n2 rc $?"; tail -5 gpurun_out/bench_n2_shared.err
