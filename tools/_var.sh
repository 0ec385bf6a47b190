b() { python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v.json 2>gpurun_out/bench_v.err; python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); r=d['roofline']
print('$1 value',round(d['value']/1e6,1),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,1),'vote_ms',round(r['kernel_ms_per_solve'],4))" || tail -3 gpurun_out/bench_v.err; }
for v in "-DRV_NP=2" "-DRV_NP=4" "-DRV_PRED=1" "-DRV_NP=4 -DRV_PRED=1"; do
RV_NVCC_EXTRA="$v" python paper_2502_06337_b200/build.py --force > /dev/null
b "$v"
python -m pytest tests/test_gpu_parity.py -x -q -k "grid or accumulate" 2>&1 | tail -1
done
