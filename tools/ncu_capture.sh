# GPU box: one ncu --set full capture per hot kernel of the config-2 bench
# (frame 5, pyramid level 0) + the launch list; reports under gpurun_out/.
CMD="python bench.py --frames 10 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1
for spec in "k_icp_reduce:91" "k_raycast_march:14" "k_raycast_lift_coop:14" "k_integrate_hashed:5"; do
  k=${spec%%:*}; s=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -f -o gpurun_out/prof_$k $CMD \
    > gpurun_out/ncu_$k.log 2>&1; echo "$k=$?"
done
