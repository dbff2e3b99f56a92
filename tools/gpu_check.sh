# GPU box: the -m gpu suite (optionally a -k filter in $K), then the config-2 bench.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu.log | grep -E "passed|failed|FAIL|Error|s call" | head -30
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1)); print({k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}); print('per_frame', d['per_frame'])"
