#!/bin/bash
# A/B of the Cholesky list's locality bucket (ELMDDM_CHOL_LOCALITY, us) on config 4: bench
# alternating on one box, then k_chol_ll DRAM reads / L2 hit rate under ncu for each value.
#   bash tools/chol_locality_ab.sh "0 500 1500 5000"
set -u
VALS=${1:-"0 500 1500 5000"}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/cl
bash tools/ab_env.sh ELMDDM_CHOL_LOCALITY "$VALS" 4 2
for w in $VALS; do
  ELMDDM_CHOL_LOCALITY=$w timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:k_chol_ll --csv python tools/profile_step.py --config 4 --steps 1 > gpurun_out/cl/ncu_$w.csv 2>&1
done
