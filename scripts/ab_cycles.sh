M=sm__cycles_elapsed.max,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second
for f in build/ab/*.so; do
  GESR_LIB=$PWD/$f timeout 300 python scripts/kbench.py --iters 1 --out-dtype bf16 > /dev/null 2>&1 || { echo "$f plain failed"; continue; }
  GESR_LIB=$PWD/$f timeout 600 ncu --metrics $M --clock-control none -k regex:${AB_KERNEL:-attn_pair} -c 2 --csv python scripts/kbench.py --iters 1 --out-dtype bf16 2>/dev/null | grep -E "${AB_KERNEL:-attn_pair}" | awk -F'","' -v f=$f '{gsub(/"/,"",$NF); print f, $(NF-2), $NF}'
done
