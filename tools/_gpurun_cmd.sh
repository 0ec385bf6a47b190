python -m pytest tests -m gpu -q -x -rf 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
RV_NVCC_EXTRA="-DRV_COOP_TRACE" python paper_2502_06337_b200/build.py --force > /dev/null
python tools/coop_trace.py c3 > gpurun_out/coop_trace_c3.txt 2>&1
python paper_2502_06337_b200/build.py --force > /dev/null
python tools/timeline.py c3 dev flush 2>/dev/null | grep -E "coop|span" > gpurun_out/tl.txt
python tools/timeline.py c4 dev flush 2>/dev/null | grep -E "span" > gpurun_out/tl4.txt
