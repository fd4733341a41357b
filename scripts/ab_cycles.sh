# A/B by SM cycles (clock-independent): ncu sm__cycles_elapsed.max of the attention / projection
# kernels for every library in build/ab/ (kbench 3h, one timed iteration).
K=${AB_KERNEL:-attn_pair}
for f in build/ab/*.so; do
  GESR_LIB=$PWD/$f timeout 300 python scripts/kbench.py --iters 1 --out-dtype bf16 > /dev/null 2>&1 || { echo "$f plain run failed"; continue; }
  GESR_LIB=$PWD/$f timeout 600 ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none \
    -k regex:$K -c ${AB_LAUNCHES:-4} --csv python scripts/kbench.py --iters 1 --out-dtype bf16 2>/dev/null \
    | grep -E "sm__cycles_elapsed|gpu__time_duration" | awk -F'","' -v f=$f '{gsub(/"/,"",$NF); print f, $(NF-2), $NF}'
done
