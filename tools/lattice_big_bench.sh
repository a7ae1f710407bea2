#!/bin/bash
# The paper's Table 2 at 2 x 2 and 1 x 1 (configs 11, 12: the grid-panel path) -- tests and bench lines.
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/lb
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "grid_panel or lattice_paper_table2_large" 2>&1 | tail -1
for k in ${@:-11 12}; do
  timeout 1200 python bench.py --config $k --no-cpu-baseline --no-e2e --no-graph --steps 2 --warmup 1 > gpurun_out/lb/bench_cfg$k.json 2> gpurun_out/lb/bench_cfg$k.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/lb/bench_cfg$k.json').read().strip().splitlines()[-1]); print('cfg$k', round(d['ms_per_step'],1), 'lf', round(d['phases_ms']['local_factor'],1), 'panel', round(d['kernel_class_ms']['panel'],1), 'wy', round(d['kernel_class_ms']['gemm_qr'],1), d['rel_l2_vs_exact'])"
done
