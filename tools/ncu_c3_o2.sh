# GPU box: ncu --set full captures of the config-3 order-2 fusion and lift
# (frame 3's launch; level 0 for the lift) -> gpurun_out/prof_c3_*.ncu-rep
CMD="python bench.py --workload config3 --frames 4 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain_c3.log 2>&1 || { echo "plain run failed"; exit 1; }
for spec in "c3_integrate|k_integrate_hashed|3" "c3_lift2|k_raycast_lift2_coop|9"; do
  IFS='|' read -r lab rx sk <<< "$spec"
  ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $sk -c 1 -f \
    -o gpurun_out/prof_$lab $CMD > gpurun_out/ncu_$lab.log 2>&1; echo "$lab=$?"
done
