timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python tools/timeline.py c3 dev flush > gpurun_out/tl_dev.txt 2>&1; grep coop gpurun_out/tl_dev.txt
python tools/gpu_check.py 2>&1 | grep "c4 full device" | cut -c1-200
