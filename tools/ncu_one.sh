# GPU box: one ncu --set full capture of a single kernel of the config-2 bench.
# usage: LAB=name RX=regex SK=skip bash tools/ncu_one.sh
CMD="python bench.py --frames 10 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$RX" -s $SK -c 1 -f \
  -o gpurun_out/prof_$LAB $CMD > gpurun_out/ncu_$LAB.log 2>&1; echo "$LAB=$?"
