timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python tools/timeline.py c3 dev flush > gpurun_out/tl_dev.txt 2>&1; grep "plan\|span" gpurun_out/tl_dev.txt
