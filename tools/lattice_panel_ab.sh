#!/bin/bash
# Panel kind on the paper's lattice rows (configs 9, 10): default vs 8-CTA cluster panels.
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in 9 10; do
  for p8 in 0 1; do
    ELMDDM_PANEL8=$p8 ELMDDM_PANEL_CLUSTER=$p8 timeout 600 python bench.py --config $k --no-cpu-baseline --no-e2e --no-graph --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$k panel8=$p8', round(d['ms_per_step'],2), 'lf', round(d['phases_ms']['local_factor'],2), 'panel', round(d['kernel_class_ms']['panel'],2), 'wy', round(d['kernel_class_ms']['gemm_qr'],2), d['rel_l2_vs_exact'])"
  done
done
