exec > gpurun_out/dcg.log 2>&1
for lib in default ab; do
if [ $lib = ab ]; then export RVK_LIB_PATH=$PWD/paper_2306_17801_b200/lib_ab/librvk.so; fi
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_spmv_tma -s 60 -c 20 --csv python scripts/dcg_time.py 2>/dev/null | grep -E "SpmvOp<0, 0>" | python -c "
import sys,csv,collections
d=collections.defaultdict(list)
for r in csv.reader(sys.stdin):
    if len(r)>5: d['dcg' if 'Dcg' in r[4] else 'cg'].append(float(r[-1]))
print('$lib', {k:(len(v), round(sum(v)/len(v)/1000,1)) for k,v in d.items()})
"
done
