# GPU box: default bench + config-3 bench, logs under gpurun_out/
set -x
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log
timeout 1200 python bench.py --workload config3 --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo bench3=$?
tail -3 gpurun_out/bench_c3.log
