python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(round(d['ms_per_step'],4), d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
python tools/host_overhead.py 2>&1 | tail -2
