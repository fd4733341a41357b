for rep in 1 2; do for m in fork kv serial; do
echo "== $m $rep"; GESR_HMA_ORDER=$m timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['step_roofline']['kv_ms'], d['step_roofline']['tasa_ms'], d['step_roofline']['hma_ms'], d['clocks']['sm_mhz'])"
done; done
