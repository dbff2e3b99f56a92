# GPU box: one ncu --set full capture (+ the FP64 instruction counts) per hot
# kernel of the config-2 bench (frame 5; level 0 for the per-level kernels),
# and the launch list; reports under gpurun_out/.
CMD="python bench.py --frames 10 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1
FP64="smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"
# label|kernel regex|matching launches to skip (frame 5's level-0 launch; bench's first run)
for spec in "k_icp_level|k_icp_level|14" "k_raycast_march|^k_raycast_march$|4" "k_raycast_march_seg|k_raycast_march_seg|8" \
            "k_raycast_lift_coop|k_raycast_lift_coop|14" "k_integrate_hashed|k_integrate_hashed|5" \
            "k_bilateral|k_bilateral|5"; do
  IFS='|' read -r lab rx sk <<< "$spec"
  ncu --set full --metrics $FP64 --clock-control none --import-source on -k "regex:$rx" -s $sk -c 1 -f \
    -o gpurun_out/prof_$lab $CMD > gpurun_out/ncu_$lab.log 2>&1; echo "$lab=$?"
done
