# time attention variants (built into build/var/) with kbench; GESR_ATTN_PAIR selects the kernel
for f in build/var/*.so; do
  for pair in 0 1; do echo "== $f pair=$pair"; GESR_ATTN_PAIR=$pair GESR_LIB=$PWD/$f timeout 300 python scripts/kbench.py --iters 5; done
done
