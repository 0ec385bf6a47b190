# Copy a tools/profile_round.sh bundle (gpurun_out/prof) into profiles/<round> and regenerate the summary.
# usage: bash tools/refresh_profiles.sh r2
set -e
R=${1:-r2}
P=profiles/$R
mkdir -p $P
cp gpurun_out/prof/bench.json $P/bench_${R}_c3.json
cp gpurun_out/prof/bench_ref.json $P/bench_ref_${R}.json
cp gpurun_out/prof/launches.csv $P/launches_${R}.csv
cp gpurun_out/prof/vote_full.ncu-rep $P/vote_banded_${R}.ncu-rep
if [ -f gpurun_out/prof/secondary.ncu-rep ]; then
  cp gpurun_out/prof/secondary.ncu-rep $P/secondary_${R}.ncu-rep
  python tools/summarize_profiles.py --kernels $P/secondary_${R}.ncu-rep > $P/SECONDARY_${R}.txt
fi
[ -f gpurun_out/prof/timeline_c3.txt ] && grep -v Warn gpurun_out/prof/timeline_c3.txt | grep -v _warn_once > $P/timeline_c3_device.txt
[ -f gpurun_out/prof/timeline_c3_host.txt ] && grep -v Warn gpurun_out/prof/timeline_c3_host.txt | grep -v _warn_once > $P/timeline_c3_e2e.txt
[ -f gpurun_out/prof/io_bench.json ] && cp gpurun_out/prof/io_bench.json $P/io_bench_${R}.json
[ -f gpurun_out/prof/pytest_gpu.log ] && tail -3 gpurun_out/prof/pytest_gpu.log > $P/pytest_gpu_${R}.txt
[ -f gpurun_out/prof/gpu_check.log ] && cut -c1-600 gpurun_out/prof/gpu_check.log > $P/gpu_check_${R}.txt
[ -f gpurun_out/prof/config_table.json ] && cp gpurun_out/prof/config_table.json $P/config_table_${R}.json && grep -v '^{' gpurun_out/prof/config_table.err > $P/config_table_${R}.txt
[ -f gpurun_out/prof/shard_probe.txt ] && grep -v Warn gpurun_out/prof/shard_probe.txt > $P/shard_probe_${R}.txt
python tools/summarize_profiles.py --json $P/vote_banded_${R}.ncu-rep | sed "s#\"source\": \"vote_banded_${R}.ncu-rep\"#\"source\": \"$P/vote_banded_${R}.ncu-rep\"#" > $P/vote_kernel_ncu.json
{ echo "# Round $R measurement bundle (tools/profile_round.sh on one B200; see DESIGN.md section 6)"
  echo "# launch list = ncu of 'python bench.py --steps 2 --warmup 3 --no-cpu' (device solves AND pipelined e2e"
  echo "# solves, whose vote runs in 4 chunks from pinned input: per-launch averages mix both; shares are what matter)"
  python tools/summarize_profiles.py $P/launches_${R}.csv $P/vote_banded_${R}.ncu-rep; } > $P/SUMMARY_${R}.txt
echo refreshed
