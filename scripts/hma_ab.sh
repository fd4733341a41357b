for rep in 1 2; do for v in ${HMA_VARIANTS:-hold hw hwn}; do GESR_LIB=build/ab/$v.so timeout 120 python scripts/hma_ab.py; done; done
