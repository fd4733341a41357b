# K-HMA session: parity tests, interleaved A/B timing of library variants (build/ab/*.so) on
# configs 3h and 5, and one ncu --set full capture of the current kernel.  TAG names the outputs.
TAG=${TAG:-hma}
mkdir -p gpurun_out
[ "${TESTS:-1}" = 1 ] && timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "hma or HMA or configs or smoke" > gpurun_out/hma_tests_$TAG.log 2>&1; echo exit=$? >> gpurun_out/hma_tests_$TAG.log
for cfg in 3h 5; do for rep in 1 2 3; do for f in build/ab/*.so; do
  GESR_LIB=$PWD/$f timeout 120 python scripts/hma_ab.py $cfg >> gpurun_out/hma_ab_$TAG.txt 2>&1
done; done; done
[ "${NCU:-1}" = 1 ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:hma_kernel -s 3 -c 1 -o gpurun_out/hma_$TAG python scripts/hma_ab.py 3h > gpurun_out/hma_ncu_$TAG.log 2>&1
echo done
