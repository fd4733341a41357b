# A/B: fused Q projection (default) vs the separate projection kernel (GESR_FUSED_Q=0), interleaved
CFG=${CFG:-3h}
for i in 1 2 3; do
  for f in 1 0; do
    GESR_FUSED_Q=$f timeout 300 python bench.py --config $CFG --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg=$CFG fused=$f', round(d['ms_per_step'],3), 'tasa', round(d['step_roofline']['tasa_ms'],3), 'kv', round(d['step_roofline']['kv_ms'],3), 'hma', round(d['step_roofline']['hma_ms'],3), 'clk', d['clocks']['sm_mhz'])"
    sleep 2
  done
done
