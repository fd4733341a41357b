# Small-config A/B (launch-bound configs 1, 2, 4) of the libraries in build/ab/, after the GPU tests.
mkdir -p gpurun_out
[ "${TESTS:-1}" = 1 ] && { timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_${TAG:-s}.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests_${TAG:-s}.log; }
for rep in 1 2; do for c in ${CFGS:-4 1 2}; do for f in build/ab/*.so; do
  echo "$(basename $f) cfg=$c $(GESR_LIB=$PWD/$f timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])')" >> gpurun_out/small_ab_${TAG:-s}.txt
done; done; done
for f in build/ab/*.so; do GESR_LIB=$PWD/$f timeout 200 python scripts/small_timeline.py --config 4 --tag $(basename $f .so) >> gpurun_out/small_tl_${TAG:-s}.txt 2>&1; done
