for c in 1024 512 256; do for cfg in 3h 5; do GESR_HMA_CHUNK=$c python scripts/hma_ab.py $cfg | sed "s/^/chunk=$c cfg=$cfg /"; done; done
