# interleaved A/B: HMA chunk variants (hma_ab.py) and K-PROJ epilogue variants (kbench.py)
for rep in 1 2; do
  for v in old c512 c1024; do GESR_LIB=build/ab/$v.so timeout 120 python scripts/hma_ab.py; done
  for v in base pld2; do echo "== $v"; GESR_LIB=build/ab/$v.so timeout 200 python scripts/kbench.py --iters 10 --out-dtype bf16; done
done
