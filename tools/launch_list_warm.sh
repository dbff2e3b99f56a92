CMD="python bench.py --frames 10 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 2000 --csv --log-file gpurun_out/launches_warm.csv $CMD > gpurun_out/ncu_ll.log 2>&1; echo ncu=$?
