mkdir -p gpurun_out
for o in row pencil; do
RVK_TILE_ORDER=$o timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_spmv_tma -s 4 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config 7pt768 > gpurun_out/ncu768_$o.csv 2> gpurun_out/ncu768_$o.err; echo "$o rc $?"; grep -E "dram__|lts__|gpu__time|l1tex" gpurun_out/ncu768_$o.csv | cut -d, -f13-16
done
