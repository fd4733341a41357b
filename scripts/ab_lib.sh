# A/B of library variants (build/ab/*.so via scripts/mkvar.sh) on bench.py, interleaved
CFG=${CFG:-3h}
for rep in $(seq ${AB_REPS:-3}); do
  for f in build/ab/*.so; do
    GESR_LIB=$PWD/$f timeout 300 python bench.py --config $CFG --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],3), 'tasa', round(d['step_roofline']['tasa_ms'],3), 'kv', round(d['step_roofline']['kv_ms'],3), 'clk', d['clocks']['sm_mhz'])"
    sleep 1
  done
done
