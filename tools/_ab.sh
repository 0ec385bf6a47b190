for cum in 0,1,3,8,16 0,1,3,7,12,16 0,1,3,6,10,16 0,1,2,4,7,11,16 0,1,3,6,11,16 0,1,3,8,16 0,1,3,7,12,16; do
RV_PIPE_CUM=$cum python bench.py --steps 20 --warmup 3 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$cum', round(d['ms_per_step'],4), d['e2e']['value'])"
done
