# round-1 GPU session script: tests, bench, launch list, one full ncu capture (run via gpurun)
set -x
TAG=${TAG:-r1}
timeout 400 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_exit=$? >> gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" = "1" ]; then
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|proj_kernel|hma_kernel|build_units" --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_pair|proj_kernel|hma_kernel" -s 4 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
fi
echo all_done
if [ "${NCU_EXTRA:-0}" = "1" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stu_$TAG.csv python scripts/stu_bench.py --iters 2 > gpurun_out/ncu_stu_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hist_$TAG.csv python scripts/history_bench.py --iters 2 > gpurun_out/ncu_hist_$TAG.log 2>&1
timeout 120 python scripts/stu_bench.py > gpurun_out/stu_$TAG.json 2>&1
timeout 120 python scripts/history_bench.py > gpurun_out/hist_$TAG.json 2>&1
fi
echo extra_done
