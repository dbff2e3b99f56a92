timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest=$rc
tail -5 gpurun_out/pytest_gpu.log
[ $rc -eq 0 ] || exit 1
timeout 900 python bench.py --workload config5 > gpurun_out/bench_c5.log 2>&1; echo bench5=$?
tail -2 gpurun_out/bench_c5.log | cut -c1-1500
