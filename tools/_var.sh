b() { python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_v.json 2>gpurun_out/bench_v.err; python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); r=d['roofline']
print('$1 value',round(d['value']/1e6,1),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,1),'vote_k',round(r['kernel_ms_per_solve'],4))" || tail -3 gpurun_out/bench_v.err; }
for v in "-DRV_STEP_UNROLL=1" "-DRV_STEP_UNROLL=2" "-DRV_STEP_UNROLL=1" "-DRV_STEP_UNROLL=2"; do
RV_NVCC_EXTRA="$v" python paper_2502_06337_b200/build.py --force > /dev/null
b "$v"
done
