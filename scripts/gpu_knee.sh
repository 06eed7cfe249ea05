mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
run() { # tag env config
  env $2 timeout 900 ncu --metrics $M --clock-control none -k regex:k_spmv_tma -s 4 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config $3 > gpurun_out/knee_$1.csv 2>/dev/null
  echo "$1 $(grep -v '^==' gpurun_out/knee_$1.csv | grep -v '^{' | awk -F'","' 'NR>1{printf "%s=%s ", $(NF-2), $NF}')"
}
run 384row RVK_TILE_ORDER=row 7pt384
run 512row RVK_TILE_ORDER=row 7pt512
run 768c40 RVK_CHUNK_MB=40 7pt768
run 768c16 "RVK_CHUNK_MB=16 RVK_CHUNK_MIN_TILES=64" 7pt768
run 768c8 "RVK_CHUNK_MB=8 RVK_CHUNK_MIN_TILES=32" 7pt768
