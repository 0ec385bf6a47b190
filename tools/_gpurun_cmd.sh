python -m pytest tests -m gpu -q -x -rf 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python tools/fuzz_estimate.py 9 180 > gpurun_out/fuzz_est.txt 2>&1
python tools/config_table.py > gpurun_out/ct.json 2> gpurun_out/ct_multi.txt
RV_COOP_MULTI=0 python tools/config_table.py > gpurun_out/ct0.json 2> gpurun_out/ct_single.txt
