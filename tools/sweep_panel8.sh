set -u
mkdir -p gpurun_out/sw
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sw/build.log 2>&1
for P8 in 0 1; do
  for spec in "2 1" "4 8" "4 16" "3 4" "3 8"; do
    ELMDDM_PANEL8=$P8 ELMDDM_PANEL_CLUSTER=$P8 timeout 300 python tools/rank_slab.py $spec >> gpurun_out/sw/slab_p8_$P8.txt 2>&1
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trsm_w -c 1 -o gpurun_out/sw/full_k_trsm_w python tools/profile_step.py --config 4 --steps 1 > gpurun_out/sw/ncu_trsm.log 2>&1
echo done
