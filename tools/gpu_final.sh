# GPU box: the round's measurement set — smoke, every bench workload (GPU arm
# and --impl reference), the expected-scaling model, the FP64 peak, the
# launch list and the ncu captures of the config-2 hot kernels.
# Logs under gpurun_out/final/ (and the ncu reports under gpurun_out/).
mkdir -p gpurun_out/final tools/_build
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke=$?
for wl in config2 config1 config3 config4 config5 reloc surfel; do
  timeout 1200 python bench.py --workload $wl > gpurun_out/final/bench_$wl.log 2>&1; echo $wl=$?
  timeout 900 python bench.py --workload $wl --impl reference > gpurun_out/final/ref_$wl.log 2>&1; echo ref_$wl=$?
done
timeout 900 python tools/scaling_model.py > gpurun_out/final/scaling_model.json 2> gpurun_out/final/scaling_model.err; echo scaling=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/_build/fp64_peak && \
  tools/_build/fp64_peak > gpurun_out/final/fp64_peak.json; echo fp64=$?
bash tools/ncu_capture.sh
python tools/ncu_traffic.py config2 r02 > gpurun_out/final/traffic.log 2>&1; echo traffic=$?
bash tools/ncu_c3_o2.sh
python tools/ncu_traffic.py config3 r02 > gpurun_out/final/traffic_c3.log 2>&1; echo traffic_c3=$?
