# GPU box: one ncu --set full capture per hot kernel of the config-2 bench
# (frame 5; level 0 unless noted) + the launch list; reports under gpurun_out/.
CMD="python bench.py --frames 10 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1
# label|kernel regex|matching launches to skip
for spec in "k_icp_reduce|k_icp_reduce|91" "k_icp_solve_t|k_icp_solve_t|91" "k_raycast_march|k_raycast_march<|4" \
            "k_raycast_march_seg|k_raycast_march_seg|9" "k_raycast_lift_coop|k_raycast_lift_coop|14" \
            "k_integrate_hashed|k_integrate_hashed|5"; do
  IFS='|' read -r lab rx sk <<< "$spec"
  ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $sk -c 1 -f -o gpurun_out/prof_$lab $CMD \
    > gpurun_out/ncu_$lab.log 2>&1; echo "$lab=$?"
done
