lscpu | grep -E "Model name|^CPU\(s\)|MHz" | head -4
for i in 1 2 3; do python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('20 steps', d['value'], d['ms_per_step'])"
python bench.py --config 3 --mlmc | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mlmc', d['value'], d['wall_s'])"
