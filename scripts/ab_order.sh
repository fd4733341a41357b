# interleaved A/B of where HMA runs in the step (bench --hma-order)
for rep in $(seq ${AB_REPS:-3}); do
  for o in fork kv serial; do
    timeout 300 python bench.py --config ${CFG:-3h} --hma-order $o --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['step_roofline']; print('$o', round(d['ms_per_step'],3), 'kv', round(r['kv_ms'],3), 'tasa', round(r['tasa_ms'],3), 'hma', round(r['hma_ms'],3), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])"
    sleep 1
  done
done
