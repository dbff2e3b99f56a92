# GPU box: parity tests then the default bench (logs under gpurun_out/)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest=$rc
tail -5 gpurun_out/pytest_gpu.log
[ $rc -eq 0 ] || exit 1
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms/step', round(d['ms_per_step'],2)); print({k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
