# attention A/B: GPU parity subset for the current library, then base-clock ncu of the pair kernel
# (build/ab/*.so) on configs 3h, 3 and 5
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${PYK:-parity or configs or sweep or history or nro}" > gpurun_out/attn_tests_${TAG}.log 2>&1; echo exit=$? >> gpurun_out/attn_tests_${TAG}.log
for c in ${CFGS:-3h 3 5}; do CFG=$c AB_REPS=${AB_REPS:-1} KREGEX=attn_pair bash scripts/ab_ncu.sh >> gpurun_out/attn_abn_${TAG}.txt 2>&1; done
echo done
