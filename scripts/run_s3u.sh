# level setup on the device
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "device_setup" > gpurun_out/pytest_s3u.log 2>&1; echo "pytest $?"; tail -15 gpurun_out/pytest_s3u.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s3u_c4.json 2>gpurun_out/s3u_c4.err; python -c "
import json; d=json.load(open('gpurun_out/s3u_c4.json')); print(round(d['value'],1), d['config'].get('setup_device'))"; tail -3 gpurun_out/s3u_c4.err
