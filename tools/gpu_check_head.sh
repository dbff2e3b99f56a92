# GPU box: confirm HEAD — smoke, the full GPU suite, config 2 and config 3 bench lines.
mkdir -p gpurun_out/head
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/head/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/head/pytest_gpu.log 2>&1; echo pytest=$?
for wl in config2 config3; do
  timeout 900 python bench.py --workload $wl > gpurun_out/head/bench_$wl.log 2>&1; echo $wl=$?
done
