python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for g in 1 0 1 0; do RV_GRAPHS=$g python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('graphs=$g', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['e2e']['value'])"; done
python tools/timeline.py c3 host flush > gpurun_out/tl_host.txt 2>&1; grep -v Warn gpurun_out/tl_host.txt | grep -v _warn | head -8; tail -1 gpurun_out/tl_host.txt
