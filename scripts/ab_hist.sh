for rep in 1 2 3; do for v in base hist; do echo "== $v"; GESR_LIB=build/ab/$v.so timeout 200 python scripts/kbench.py --iters 10 --out-dtype bf16; done; done
