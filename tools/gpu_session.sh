#!/bin/bash
# One gpurun session: GPU tests, smoke, bench (cfg3), ncu launch list of the same step.
# usage (from the repo root on the box): bash tools/gpu_session.sh TAG [what...]
#   what: tests smoke bench launches full:<kernel-regex> bench<k>
set -u
TAG=${1:-run}; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/nvsmi.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo BUILD FAILED; tail -30 "$OUT/build.log"; exit 1; }
for w in "$@"; do
  case "$w" in
    tests)
      timeout 1500 python -m pytest tests -m gpu -q > "$OUT/tests.log" 2>&1; echo "tests exit $?" | tee -a "$OUT/summary.txt"
      tail -5 "$OUT/tests.log";;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" | tee -a "$OUT/summary.txt";;
    bench)
      timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench exit $?" | tee -a "$OUT/summary.txt"
      cat "$OUT/bench.json";;
    bench[0-9])
      k=${w#bench}
      timeout 900 python bench.py --config "$k" --no-cpu-baseline > "$OUT/bench_cfg$k.json" 2> "$OUT/bench_cfg$k.err"; echo "bench cfg$k exit $?" | tee -a "$OUT/summary.txt"
      cat "$OUT/bench_cfg$k.json";;
    cfg:*)
      k=${w#cfg:}
      timeout 1200 python bench.py --config "$k" --no-cpu-baseline --no-e2e --steps 3 --warmup 1 > "$OUT/bench_cfg$k.json" 2> "$OUT/bench_cfg$k.err"; echo "bench cfg$k exit $?" | tee -a "$OUT/summary.txt"
      python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], d['ms_per_step'], d.get('rel_l2_vs_exact'))" "$OUT/bench_cfg$k.json";;
    nd[0-9]|strip[0-9])
      k=${w: -1}; m=3; [ "${w:0:5}" = strip ] && m=2
      timeout 900 python bench.py --config "$k" --interface-mode $m --no-cpu-baseline --no-e2e > "$OUT/bench_${w}.json" 2> "$OUT/bench_${w}.err"; echo "bench $w exit $?" | tee -a "$OUT/summary.txt"
      python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], d['ms_per_step'], d['phases_ms'], d['config'].get('interface_ordering'))" "$OUT/bench_${w}.json";;
    probe)
      timeout 300 python -c "
import json,subprocess,torch,paper_2406_15959_b200 as E
torch.cuda.init()
smi=lambda: subprocess.run(['nvidia-smi','--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active','--format=csv,noheader'],capture_output=True,text=True).stdout.strip()
r=[]
for ms in (300.0,1000.0,3000.0):
    before=smi(); t=E.solver.dmma_peak_tflops(0,ms); r.append(dict(ms=ms,tflops=t,smi_before=before,smi_after=smi()))
print(json.dumps(dict(probe='elmddm_dmma_probe (register-resident DMMA.8x8x4 loop, 148 SMs)',runs=r,gpu=subprocess.run(['nvidia-smi','--query-gpu=name,driver_version','--format=csv,noheader'],capture_output=True,text=True).stdout.strip()),indent=1))
" > "$OUT/dmma_probe.json" 2>&1; echo "probe exit $?" | tee -a "$OUT/summary.txt"; cat "$OUT/dmma_probe.json";;
    ref)
      timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/ref.json" 2> "$OUT/ref.err"; echo "ref exit $?" | tee -a "$OUT/summary.txt";;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
        --log-file "$OUT/launches.csv" python tools/profile_step.py --config ${CFG:-3} --steps 1 > "$OUT/ncu_launches.log" 2>&1
      echo "launches exit $?" | tee -a "$OUT/summary.txt"
      python tools/launches.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1; head -25 "$OUT/launches_summary.txt";;
    traffic)
      timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:k_wy_tma --csv --log-file "$OUT/traffic.csv" python tools/profile_step.py --config ${CFG:-3} --steps 1 > "$OUT/ncu_traffic.log" 2>&1
      echo "traffic exit $?" | tee -a "$OUT/summary.txt"
      python tools/traffic.py "$OUT/traffic.csv" ${CFG:-3} "$OUT/traffic_cfg${CFG:-3}.json";;
    full:*)
      spec=${w#full:}; k=${spec%%:*}; skip=2
      [ "$spec" != "$k" ] && skip=${spec#*:}
      timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$k" -s $skip -c 1 \
        -o "$OUT/full_${k//[^a-zA-Z0-9_]/_}" python tools/profile_step.py --config ${CFG:-3} --steps 1 > "$OUT/ncu_full_${k//[^a-zA-Z0-9_]/_}.log" 2>&1
      echo "full $k exit $?" | tee -a "$OUT/summary.txt";;
  esac
done
