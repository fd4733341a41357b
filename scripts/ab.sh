# A/B: alternate the libraries in build/var/ three times (same box, same process type)
for rep in 1 2 3; do
  for f in build/var/*.so; do
    echo "== $f rep=$rep"; GESR_LIB=$PWD/$f timeout 300 python scripts/kbench.py --iters 10
  done
done
