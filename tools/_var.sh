for v in "-DRV_TAIL_DIV=1000000 -DRV_TAIL_GRAB=32" "-DRV_TAIL_DIV=32 -DRV_TAIL_GRAB=8" "-DRV_TAIL_DIV=64 -DRV_TAIL_GRAB=16" "-DRV_TAIL_DIV=16 -DRV_TAIL_GRAB=8"; do
RV_NVCC_EXTRA="$v" python paper_2502_06337_b200/build.py --force > /dev/null
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_v.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_v.json'))
print('$v value',round(d['value']/1e6,1),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3),'vk',round(d['roofline']['kernel_ms_per_solve'],4))"
done
