python tools/guard_probe.py > gpurun_out/guard_probe.txt 2>&1
python -m pytest tests -m gpu -q -rf 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
bash tools/_ab.sh "" > gpurun_out/ab.log 2>&1
