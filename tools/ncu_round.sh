# Round profile evidence (one GPU): launch list of one whole-network training
# step, then a --set full capture of the largest launch (block 1, layer 15) of
# each conv kernel type and of the BN-apply kernel.  Each ncu run follows a
# plain run of the same command.
#   bash tools/ncu_round.sh [round]          SKIP_LIST=1 / SPECS="kernel:skip ..." to narrow
R=${1:-r01}
CMD="python bench.py --ncu-step --ncu-what model --no-cpu-baseline"
if [ "${SKIP_LIST:-0}" != 1 ]; then
  $CMD > gpurun_out/${R}_plain.log 2>&1 && ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_list.log 2>&1
  echo "launch list rc=$?"
fi
# forward order: block 1 first (layer 15 = 16th launch); backward order: block 3,
# 2, then 1 (block 1 layer 15 = 33rd launch of each backward kernel)
SPECS=${SPECS:-"Fwd1x1:15 Tc3x3FwdTaps:15 Tc3x3DgradHalo:32 Dgrad1x1:32 Wgrad1x1:32 Tc3x3WgradHalo:32 k_bn_apply_accumulate4:32"}
for spec in $SPECS; do
  k=${spec%%:*}; s=${spec##*:}
  $CMD > gpurun_out/${R}_plain_$k.log 2>&1 && ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k -s $s -c 1 -o gpurun_out/${R}_$k $CMD > gpurun_out/${R}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
