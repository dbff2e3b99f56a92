# Local: copy the round's measurement set (gpurun_out/final, gpurun_out/*.csv|ncu-rep)
# into profiles/ as <round>_* files; usage: bash tools/collect_final.sh r02
R=${1:-r02}
F=gpurun_out/final
for wl in config2 config1 config3 config4 config5 reloc surfel; do
  [ -s $F/bench_$wl.log ] && tail -1 $F/bench_$wl.log > profiles/${R}_bench_$wl.json
  [ -s $F/ref_$wl.log ] && tail -1 $F/ref_$wl.log > profiles/${R}_bench_reference_$wl.json
done
[ -s gpurun_out/pytest_gpu_full.log ] && cp gpurun_out/pytest_gpu_full.log profiles/${R}_pytest_gpu_full.log
cp $F/smoke.log profiles/${R}_smoke.log 2>/dev/null
cp $F/gpu.txt profiles/${R}_gpu.txt 2>/dev/null
[ -s $F/scaling_model.json ] && cp $F/scaling_model.json profiles/${R}_scaling_model.json
[ -s $F/fp64_peak.json ] && cp $F/fp64_peak.json profiles/${R}_fp64_peak.json
if [ -s gpurun_out/launches.csv ]; then
  cp gpurun_out/launches.csv profiles/${R}_ncu_launches.csv
  python tools/launches.py gpurun_out/launches.csv > profiles/${R}_ncu_launches_summary.txt
fi
