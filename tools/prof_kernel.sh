#!/bin/bash
# usage: bash tools/prof_kernel.sh TAG KERNEL_REGEX [config] [skip]
set -u
TAG=$1; K=$2; CFG=${3:-3}; SKIP=${4:-0}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
N=${K//[^a-zA-Z0-9_]/_}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s $SKIP -c 1 -o $OUT/$N \
  python tools/profile_step.py --config $CFG --steps 1 > $OUT/ncu_$N.log 2>&1; echo "ncu $K exit $?"
