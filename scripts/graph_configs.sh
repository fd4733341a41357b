# Configs 1, 2, 4 (launch-bound) eager vs --graph bench lines, and 3h under --graph.
mkdir -p gpurun_out
for c in ${CFGS:-1 2 4}; do for g in "" "--graph"; do
 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline $g > gpurun_out/bg_${c}${g}.json 2> gpurun_out/bg_${c}${g}.err
done; done
[ "${BIG:-1}" = 1 ] && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --graph > gpurun_out/bg_3h_graph.json 2> gpurun_out/bg_3h_graph.err
