# GPU box: FP64 peak microbenchmark, the default bench line, the launch list
# and the per-kernel ncu captures (tools/ncu_capture.sh); logs under gpurun_out/.
mkdir -p tools/_build gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/_build/fp64_peak && \
  tools/_build/fp64_peak > gpurun_out/fp64_peak.json; echo fp64=$?; cat gpurun_out/fp64_peak.json
bash tools/ncu_capture.sh
