# dev helper: parity tests + timing probe (+ optional ncu of the vote kernel)
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
python tools/gpu_check.py > gpurun_out/gpu_check.log 2>&1; grep -E "mismatch|inliers equal|multi|full device" gpurun_out/gpu_check.log | cut -c1-330
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_dev.json 2> gpurun_out/bench_dev.err; python -c "
import json; d=json.load(open('gpurun_out/bench_dev.json')); r=d['roofline']
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'vote_ms',r['kernel_ms_per_solve'],'frac',r['frac'],'stage',d['stage_ms'])"
if [ -n "$NCU" ]; then ncu --set full --import-source on --clock-control none -k regex:vote_banded -c 1 -f -o gpurun_out/$NCU python tools/profile_vote.py c3 1 > gpurun_out/ncu_$NCU.log 2>&1; echo ncu_rc=$?; fi
