timeout 600 python gpurun_out/iters.py 2>&1 | tail -20
timeout 900 python -m pytest tests -m gpu -x -v -p no:cacheprovider > gpurun_out/pytest2.log 2>&1; echo "pytest exit $?"
grep -E "PASS|FAIL|Error|error|Fatal" gpurun_out/pytest2.log | head -40
