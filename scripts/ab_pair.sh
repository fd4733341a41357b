# Parity of the CTA-pair attention path, then interleaved A/B vs the 1-CTA kernel.
GESR_ATTN_PAIR=1 timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for rep in $(seq ${AB_REPS:-3}); do
  for v in 0 1; do
    echo "== pair=$v rep=$rep"; GESR_ATTN_PAIR=$v timeout 300 python scripts/kbench.py --iters ${AB_ITERS:-10} --out-dtype bf16
  done
done
