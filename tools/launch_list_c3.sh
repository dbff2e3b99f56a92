# GPU box: warm-cache ncu launch list of a short config-3 run
CMD="python bench.py --workload config3 --frames 4 --steps 1 --warmup 0 --no-cpu"
$CMD > gpurun_out/plain_c3.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_ll_c3.log 2>&1; echo ncu=$?
