timeout 600 python scripts/debug_tma.py 0 1 2 4 6 7 8 9 10 12
