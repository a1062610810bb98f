for t in 0 1 2 3 4 5 6 7 8; do ./scripts/tma_probe.bin $t | tail -1; done
