timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?
bash tools/gpu_final.sh
