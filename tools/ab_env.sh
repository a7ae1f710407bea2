#!/bin/bash
# A/B of one environment knob on the cfg bench, alternating runs on the same box:
#   bash tools/ab_env.sh VAR "v1 v2" [config] [rounds]  -> gpurun_out/ab/<VAR>.txt
set -u
VAR=$1; VALS=$2; CFG=${3:-4}; ROUNDS=${4:-2}
mkdir -p gpurun_out/ab
for r in $(seq 1 "$ROUNDS"); do
  for v in $VALS; do
    env "$VAR=$v" timeout 600 python bench.py --config "$CFG" --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab/run.json 2> /dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab/run.json').read().strip().splitlines()[-1]); print(sys.argv[1], sys.argv[2], round(d['ms_per_step'],2), 'lf', round(d['phases_ms']['local_factor'],2), 'wy', round(d['kernel_class_ms']['gemm_qr'],2), 'schur', round(d['phases_ms']['schur_accumulate'],2), 'iface', round(d['phases_ms']['interface_factor_solve'],2), 'mhz', d['clocks']['sm_mhz'])" "$VAR=$v" "round $r" | tee -a gpurun_out/ab/$VAR.txt
  done
done
