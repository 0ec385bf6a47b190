python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for g in 1 0 1; do RV_GRAPHS=$g python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('graphs=$g', round(d['ms_per_step'],4), d['value'], d['e2e']['value'])"; done
python tools/timeline.py c3 > gpurun_out/tl_dev.txt 2>&1; grep -v Warn gpurun_out/tl_dev.txt | grep -v _warn | head -4
python tools/timeline.py c3 dev flush > gpurun_out/tl_devf.txt 2>&1; grep -v Warn gpurun_out/tl_devf.txt | grep -v _warn | head -3; tail -1 gpurun_out/tl_devf.txt
