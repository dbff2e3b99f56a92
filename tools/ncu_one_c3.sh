# GPU box: one ncu --set full capture of a config-3 kernel (LAB, RX, SK as ncu_one.sh)
CMD="python bench.py --workload config3 --frames 4 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain_c3.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$RX" -s $SK -c 1 -f \
  -o gpurun_out/prof_$LAB $CMD > gpurun_out/ncu_$LAB.log 2>&1; echo "$LAB=$?"
