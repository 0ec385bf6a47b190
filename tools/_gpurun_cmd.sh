python -m pytest tests -m gpu -q -x -rf 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
bash tools/_ab.sh "-DRV_ENTRY_RELOAD=0" "" "-DRV_ENTRY_RELOAD=0" "" > gpurun_out/ab.log 2>&1
