# A/B: alternate the libraries in ${AB_DIR:-build/ab}/ three times (same box, same process type)
for rep in $(seq ${AB_REPS:-3}); do
  for f in ${AB_DIR:-build/ab}/*.so; do
    echo "== $f rep=$rep"; GESR_LIB=$PWD/$f timeout 300 python scripts/kbench.py --iters 10 --out-dtype ${AB_DTYPE:-bf16}
  done
done
