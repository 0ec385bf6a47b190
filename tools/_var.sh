b() { python bench.py --steps 10 --warmup 3 > gpurun_out/bench_v.json 2>gpurun_out/bench_v.err; python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); r=d['roofline']
print('$1 value',round(d['value']/1e6,1),'ms',round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,1),'vote_ms',round(r['vote_ms_per_solve'],4))" || tail -3 gpurun_out/bench_v.err; }
b t640
for t in 768 832 896 1024; do
sed -i "s/constexpr int kVoteThreads = [0-9]*;/constexpr int kVoteThreads = $t;/" paper_2502_06337_b200/csrc/rv_internal.h
python paper_2502_06337_b200/build.py -v 2>&1 | grep -A2 "Function properties for.*vote_banded_kernelILb0" | grep -E "Used|spill" | tr '\n' ' '
b t$t
done
