timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest=$rc
tail -5 gpurun_out/pytest_gpu.log
[ $rc -eq 0 ] || exit 1
timeout 1500 python bench.py --workload config4 --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo bench4=$?
tail -2 gpurun_out/bench_c4.log | cut -c1-1800
