# dev A/B sweep on the GPU box: rebuild with each macro set, run a short bench, print vote-kernel time
for v in "$@"; do
RV_NVCC_EXTRA="$v" python paper_2502_06337_b200/build.py --force > /dev/null
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_v.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_v.json'))
print('[$v] ms',round(d['ms_per_step'],4),'e2e',round(d['e2e']['ms_per_step'],4),'vk',round(d['roofline']['kernel_ms_per_solve'],4),'frac',round(d['roofline']['frac'],3), 'vote_stage', round(d['stage_ms']['vote_ms'],4))"
done
