mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_pdl.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests_pdl.log
for rep in 1 2; do for c in 2 4 1 3h; do for f in build/ab/*.so; do
  echo "$(basename $f) cfg=$c $(GESR_LIB=$PWD/$f timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')" >> gpurun_out/pdl_ab.txt
done; done; done
GESR_LIB=$PWD/build/ab/a_pdl.so timeout 300 python scripts/graph_bench.py --iters 50 > gpurun_out/graph_pdl.jsonl 2>&1
GESR_LIB=$PWD/build/ab/b_nopdl.so timeout 300 python scripts/graph_bench.py --iters 50 > gpurun_out/graph_nopdl.jsonl 2>&1
