for cum in "0,1,4,10,16" "0,1,5,16" "0,2,6,16" "0,1,3,8,16" "0,1,4,10,16" "0,2,5,10,16"; do
RV_PIPE_CUM=$cum python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_v.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_v.json'))
print('cum $cum value',round(d['value']/1e6,1),'e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3))"
done
