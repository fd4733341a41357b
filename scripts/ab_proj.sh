# A/B the libraries in build/ab/ (kbench 3h); ORDERS selects GESR_PROJ_ORDER values to sweep
for rep in $(seq ${AB_REPS:-3}); do for f in build/ab/*.so; do for o in ${ORDERS:-1}; do
  echo "== $f order=$o rep=$rep"
  GESR_PROJ_ORDER=$o GESR_LIB=$PWD/$f timeout 300 python scripts/kbench.py --iters 10 --out-dtype bf16 2>&1 | tail -1
done; done; done
