timeout 1500 python scripts/cfg5_sweep.py 1e-2,3e-3,1e-3 2>&1 | grep -v "^ " | tail -14
