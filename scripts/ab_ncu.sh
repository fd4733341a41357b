# Clock-independent A/B of kernel variants: ncu at the base clock (--clock-control base), kernel
# durations and SM cycles of one bench step per library in build/ab/ (A/B decisions only; never a
# bench number)
mkdir -p gpurun_out/abn
for rep in $(seq ${AB_REPS:-2}); do
  for f in build/ab/*.so; do
    n=$(basename $f .so)
    GESR_LIB=$PWD/$f timeout 300 ncu --clock-control base --metrics gpu__time_duration.sum,sm__cycles_elapsed.max -k regex:"${KREGEX:-attn_pair|proj_kernel|hma_kernel}" --csv --log-file gpurun_out/abn/$n.csv python bench.py --config ${CFG:-3h} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
    python - gpurun_out/abn/$n.csv $n <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; iN = h.index('Kernel Name'); iM = h.index('Metric Name'); iV = h.index('Metric Value')
agg = {}
for r in rows[1:]:
    k = r[iN].split('(')[0].replace('void ', '')[-18:] + ':' + ('us' if 'duration' in r[iM] else 'cyc')
    agg.setdefault(k, []).append(float(r[iV].replace(',', '')))
print(sys.argv[2], ' '.join(f'{k}={sum(v) / len(v):.5g}' for k, v in sorted(agg.items())))
PY
  done
done
