python -m pytest tests -m gpu -q -x -rf 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python tools/timeline.py c3 dev flush 2>/dev/null | grep -E "coop|span" > gpurun_out/tl.txt
