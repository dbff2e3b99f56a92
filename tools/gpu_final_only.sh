# GPU box: the round's measurement set at HEAD, ncu summaries copied under
# gpurun_out/final/profiles, .ncu-rep files removed (gpurun copies back <= 64 MiB).
mkdir -p gpurun_out/final/profiles
bash tools/gpu_round_end.sh > gpurun_out/round_end.log 2>&1
cp profiles/r02_ncu_*.csv profiles/traffic.json gpurun_out/final/profiles/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
cat gpurun_out/round_end.log
