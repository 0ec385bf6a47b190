for g in 32 8 16 4 32 8; do RV_GRAB_SMALL=$g python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('grab=$g', round(d['e2e']['ms_per_step'],4), round(d['ms_per_step'],4))"; done
