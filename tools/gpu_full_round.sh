# GPU box: smoke, GPU tests, every bench workload, launch list + ncu captures
# of the config-2 hot kernels; logs under gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
for wl in config3 config4 config5 reloc surfel; do
  timeout 1200 python bench.py --workload $wl > gpurun_out/bench_$wl.log 2>&1; echo $wl=$?
done
bash tools/ncu_capture.sh
python tools/ncu_traffic.py > gpurun_out/traffic.log 2>&1; echo traffic=$?
