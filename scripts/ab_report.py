import json, sys, collections
cur = None; res = collections.defaultdict(list)
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line.split()[1]
    elif line.startswith("{"):
        d = json.loads(line); res[cur].append(d)
for k, v in res.items():
    f = lambda key: " ".join(f"{x[key]:.3f}" for x in v)
    print(f"{k}\n  tasa {f('tasa_ms')}\n  kv   {f('kv_ms')}\n  hma  {f('hma_ms')}\n  step {f('step_ms')}")
