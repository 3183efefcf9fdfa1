for i in 0 1 2 3 4 5; do timeout 60 ./tools/tma_probe L $i 2>&1; done
