# Round measurement set (gpurun -- 'bash scripts/measure.sh TAG [parts]'); outputs in gpurun_out/.
# parts: any of  tests bench ref cfgs mlmc levels launches ncu   (default: all)   + cesplit cfg5
TAG=${1:-x}; PARTS=${2:-"tests bench ref cfgs mlmc levels launches ncu"}
O=gpurun_out
has() { case " $PARTS " in *" $1 "*) return 0;; esac; return 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
if has tests; then
  timeout 3000 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -4 $O/${TAG}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
fi
if has bench; then
  timeout 1200 python bench.py > $O/${TAG}_cfg4.json 2> $O/${TAG}_cfg4.err; echo "bench rc=$?"
  python - <<PY
import json; d=json.load(open('$O/${TAG}_cfg4.json')); print(d['value'], d['e2e'], d['roofline'], d['pipeline_roofline']['frac'], d['cpu_baseline'], d['gpu_launches'], d['clocks'])
PY
fi
if has ref; then
  timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err; echo "ref rc=$?"; cat $O/${TAG}_ref.json
fi
if has cfgs; then
  for c in 1 2 3; do
    timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/${TAG}_c$c.json 2> $O/${TAG}_c$c.err; echo "c$c rc=$?"
    python - <<PY
import json; d=json.load(open('$O/${TAG}_c$c.json')); print(d['value'], (d.get('e2e') or {}).get('value'), d['pipeline_roofline']['frac'], (d.get('cpu_baseline') or {}).get('value'), d['roofline'].get('kernel'), d['roofline'].get('frac'), d.get('per_level'))
PY
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/${TAG}_torchrun.json 2> $O/${TAG}_torchrun.err; echo "torchrun rc=$?"; head -c 300 $O/${TAG}_torchrun.json; echo
fi
if has mlmc; then
  timeout 900 python bench.py --config 3 --mlmc > $O/${TAG}_mlmc.json 2> $O/${TAG}_mlmc.err; echo "mlmc rc=$?"; head -c 800 $O/${TAG}_mlmc.json; echo
fi
if has levels; then
  # kernel-class shares of config 3's small levels + an ncu capture of the CTA-resident solver (16^2)
  timeout 600 python scripts/level_breakdown.py 0,1,2,3 > $O/${TAG}_levels.json 2> $O/${TAG}_levels.err; echo "levels rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_pcg -s 3 -c 1 -o $O/${TAG}_small_pcg16 python scripts/level_breakdown.py 0 > $O/${TAG}_ncu_small.log 2>&1; tail -1 $O/${TAG}_ncu_small.log
  python scripts/ncu_summary.py $O/${TAG}_small_pcg16.ncu-rep 8 > $O/${TAG}_small_pcg16_ncu.txt 2>&1
  python scripts/ncu_stalls.py $O/${TAG}_small_pcg16.ncu-rep >> $O/${TAG}_small_pcg16_ncu.txt 2>&1
  python scripts/ncu_lines.py $O/${TAG}_small_pcg16.ncu-rep 20 >> $O/${TAG}_small_pcg16_ncu.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f $O/${TAG}_small_pcg16.ncu-rep
fi
if has cfg5; then
  timeout 2400 python scripts/cfg5_sweep.py > $O/${TAG}_cfg5.log 2> $O/${TAG}_cfg5.err; echo "cfg5 rc=$?"; cp $O/cfg5_sweep.json $O/${TAG}_cfg5_sweep.json
fi
CMD="python bench.py --steps 1 --warmup 1 --batch 8 --no-cpu-baseline --no-e2e"
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/${TAG}_cfg4_launches.csv $CMD > $O/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
fi
if has ncu; then
  # --set full captures of the top kernels at the 2048^2 solve (batch 8), selected by their NVTX range
  # (OSC_NVTX=1: every kernel-class scope is a range "<class>:<grid>"; OSC_LEVEL_STATS=1 names levels)
  for cls in "pcg_update:2048" "mg_smooth_up_r.L0:2048" "mg_restrict_r.L0:2048" "mg_up.L1:2048" "mg_down.L1:2048" "mg_setup.galerkin.L0:2048"; do
    f=$(echo $cls | tr ':.' '__')
    OSC_NVTX=1 OSC_LEVEL_STATS=1 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "$cls/" -s 2 -c 1 -o $O/${TAG}_$f $CMD > $O/${TAG}_ncu_$f.log 2>&1; tail -1 $O/${TAG}_ncu_$f.log
    python scripts/ncu_summary.py $O/${TAG}_$f.ncu-rep 14 > $O/${TAG}_${f}_ncu.txt 2>&1
    python scripts/ncu_stalls.py $O/${TAG}_$f.ncu-rep >> $O/${TAG}_${f}_ncu.txt 2>&1
    [ -n "$KEEP_REP" ] || rm -f $O/${TAG}_$f.ncu-rep   # gpurun_out/ returns at most 64 MiB
  done
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:ce_ -c 2 -o $O/${TAG}_ce python bench.py --config 2 --batch 32 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/${TAG}_ncu_ce.log 2>&1; tail -1 $O/${TAG}_ncu_ce.log
  python scripts/ncu_summary.py $O/${TAG}_ce.ncu-rep 14 > $O/${TAG}_ce_ncu.txt 2>&1
  python scripts/ncu_stalls.py $O/${TAG}_ce.ncu-rep > $O/${TAG}_ce_stalls.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f $O/${TAG}_ce.ncu-rep
fi
if has cesplit; then
  timeout 600 python scripts/ce_split.py > $O/${TAG}_ce_split.json 2> $O/${TAG}_ce_split.err; echo "ce_split rc=$?"; cat $O/${TAG}_ce_split.json
fi
ls -la $O | tail -40
