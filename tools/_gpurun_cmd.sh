python tools/timeline.py c4 dev flush api > gpurun_out/tl4_api.txt 2>&1
