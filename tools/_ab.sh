timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for g in 1 0 1; do RV_BULK=$g python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('bulk=$g', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['roofline']['kernel_ms_per_solve'])"; done
cp _variants/bulk516_trace.so paper_2502_06337_b200/_lib/librotavote_b200.so
for g in 1 0; do echo "== bulk=$g"; RV_BULK=$g python tools/vote_trace.py 2>&1 | tail -5 | sed -E 's/start max=[0-9.]+ init med=[0-9.]+ //'; done
cp _variants/bulk516.so paper_2502_06337_b200/_lib/librotavote_b200.so
