exec > gpurun_out/dcg.log 2>&1
for i in 1 2; do
timeout 300 python scripts/dcg_time.py 2>&1 | head -1 | sed "s/^/own /"
RVK_LIB_PATH=$PWD/paper_2306_17801_b200/lib_ab/librvk.so timeout 300 python scripts/dcg_time.py 2>&1 | head -1 | sed "s/^/no-own /"
done
