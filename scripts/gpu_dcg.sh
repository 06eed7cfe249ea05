exec > gpurun_out/dcg.log 2>&1
for st in 0 262144 524288 1048576 0; do
echo stagger $st
RVK_WIN_STAGGER=$st timeout 300 python scripts/dcg_time.py 256x256x256 2>&1 | head -1
RVK_WIN_STAGGER=$st timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"xfix|spmv" -c 6 python scripts/dcg_time.py 2>&1 | grep -E "gpu__time_duration" | tr -s ' ' | cut -d' ' -f4 | tr '\n' ' '; echo
done
