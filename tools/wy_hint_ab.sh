#!/bin/bash
# A/B of the evict-first L2 hints of the trailing update's phase 3 (ELMDDM_WY_HINT3) on config 4:
# alternating bench runs, then k_wy_tma DRAM bytes under ncu for each setting.
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/wh
ELMDDM_WY_HINT3=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "chunk_order or end_to_end_u_parity" 2>&1 | tail -1
bash tools/ab_env.sh ELMDDM_WY_HINT3 "0 1" 4 3
for h in 0 1; do
  ELMDDM_WY_HINT3=$h timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_wy_tma --csv --log-file gpurun_out/wh/traffic_$h.csv python tools/profile_step.py --config 4 --steps 1 > /dev/null 2>&1
  python tools/traffic.py gpurun_out/wh/traffic_$h.csv 4 gpurun_out/wh/traffic_$h.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('gpurun_out/wh/traffic_$h.json')); print('hint', $h, d['dram_read_bytes_per_launch'], d['dram_write_bytes_per_launch'], d['ncu_ms_per_launch'])"
done
