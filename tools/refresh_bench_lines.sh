#!/bin/bash
# Re-measure the non-headline bench lines (README "Results") with the current code.
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/rl
for k in ${@:-2 3 5 6 7 8 9 10}; do
  timeout 900 python bench.py --config $k --no-cpu-baseline > gpurun_out/rl/bench_cfg$k.json 2> gpurun_out/rl/bench_cfg$k.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/rl/bench_cfg$k.json').read().strip().splitlines()[-1]); print('cfg$k', round(d['ms_per_step'],2), round(d['value'],1), d['rel_l2_vs_exact'], d['clocks']['sm_mhz'])"
done
