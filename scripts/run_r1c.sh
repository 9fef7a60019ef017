timeout 600 python scripts/iters.py 64 256 1024 2048 2>&1 | tail -20
