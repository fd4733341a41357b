for rep in 1 2; do for dt in f32 bf16; do echo "== out=$dt rep=$rep"; timeout 300 python scripts/kbench.py --iters 10 --out-dtype $dt; done; done
