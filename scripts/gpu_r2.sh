# round-2 GPU session: tests, smoke, bench (headline + config 5), timeline, ncu launch list and
# one full ncu capture of the step's kernels.  Knobs: TAG, TESTS=0/1, NCU=0/1, EXTRA=0/1
set -x
TAG=${TAG:-r2}
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/gpu_tests_$TAG.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo exit=$? >> gpurun_out/smoke_$TAG.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_exit=$? >> gpurun_out/bench_$TAG.err
if [ "${EXTRA:-1}" = "1" ]; then
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench5_$TAG.json 2> gpurun_out/bench5_$TAG.err; echo bench_exit=$? >> gpurun_out/bench5_$TAG.err
timeout 300 python scripts/step_timeline.py --tag $TAG > gpurun_out/step_timeline_$TAG.json 2> gpurun_out/step_timeline_$TAG.err
fi
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|proj_kernel|hma_kernel|build_units" --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_pair|proj_kernel|hma_kernel" -s 4 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
fi
if [ -n "${POST:-}" ]; then bash -c "$POST" > gpurun_out/post_$TAG.log 2>&1; fi
echo all_done
