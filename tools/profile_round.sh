# Round-end measurement bundle (run under gpurun on ONE B200): bench line, reference arm,
# ncu launch list of the bench command, ncu --set full of the vote kernel. Outputs in gpurun_out/prof/.
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof/bench_ref.json 2> gpurun_out/prof/bench_ref.err; echo ref_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/prof/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
ncu --set full --import-source on --clock-control none -k regex:vote_banded -c 1 -f -o gpurun_out/prof/vote_full \
    python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/prof/ncu_full.log 2>&1; echo ncu_full_rc=$?
ncu --set full --import-source on --clock-control none -k "regex:preprocess_kernel|plan_kernel|vote_reduce|coop_refine|vote_angles|peak_angle" \
    -c 6 -f -o gpurun_out/prof/secondary python tools/profile_vote.py c3 1 > gpurun_out/prof/ncu_secondary.log 2>&1; echo ncu_secondary_rc=$?
python tools/timeline.py c3 dev flush > gpurun_out/prof/timeline_c3.txt 2>&1
python tools/timeline.py c3 host flush > gpurun_out/prof/timeline_c3_host.txt 2>&1
python tools/gpu_check.py > gpurun_out/prof/gpu_check.log 2>&1; echo gpu_check_rc=$?
python tools/io_bench.py > gpurun_out/prof/io_bench.json 2> gpurun_out/prof/io_bench.err; echo io_bench_rc=$?
python -m pytest tests -m gpu -q > gpurun_out/prof/pytest_gpu.log 2>&1; echo pytest_rc=$?
python tools/config_table.py > gpurun_out/prof/config_table.json 2> gpurun_out/prof/config_table.err; echo config_table_rc=$?
python tools/shard_probe.py > gpurun_out/prof/shard_probe.txt 2>&1; echo shard_probe_rc=$?
