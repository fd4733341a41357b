# time attention variants (built into build/var/) with kbench
for f in build/var/*.so; do echo "== $f"; GESR_LIB=$PWD/$f timeout 300 python scripts/kbench.py --iters 5; done
