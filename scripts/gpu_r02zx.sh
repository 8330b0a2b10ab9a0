#!/bin/bash
# final-state ncu of the F3 / F4 kernels (one launch each) + their launch lists
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zx.log 2>&1
for k in k_tr_gather k_tr_attn_bwd k_tr_seg_piece k_tr_attn_fwd; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_f4_gdelt_$k python scripts/exp_train_stage.py gdelt 16000 0 train > gpurun_out/ncu_full_f4_$k.log 2>&1
done
for k in k_apan_build k_apan_deliver; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_f3_gdelt_$k python scripts/exp_train_stage.py gdelt 16000 0 apan > gpurun_out/ncu_full_f3_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_train_gdelt.csv python scripts/exp_train_stage.py gdelt 12000 0 train > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_apan_gdelt.csv python scripts/exp_train_stage.py gdelt 12000 0 apan > /dev/null 2>&1
ls gpurun_out | grep -E "prof_f|final_launch"
