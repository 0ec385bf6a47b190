python tools/guard_probe.py > gpurun_out/guard_probe.txt 2>&1
python -m pytest tests -m gpu -q -x -rf 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
bash tools/_ab.sh "" > gpurun_out/ab.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:plan_kernel" -c 1 -f -o gpurun_out/plan python tools/profile_vote.py c3 1 > gpurun_out/ncu_plan.log 2>&1
