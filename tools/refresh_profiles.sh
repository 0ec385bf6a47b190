# Copy a tools/profile_round.sh bundle (gpurun_out/prof) into profiles/r1 and regenerate the summary.
set -e
P=profiles/r1
cp gpurun_out/prof/bench.json $P/bench_r1_c3.json
cp gpurun_out/prof/bench_ref.json $P/bench_ref_r1.json
cp gpurun_out/prof/launches.csv $P/launches_r1.csv
cp gpurun_out/prof/vote_full.ncu-rep $P/vote_banded_r1.ncu-rep
if [ -f gpurun_out/prof/secondary.ncu-rep ]; then
  cp gpurun_out/prof/secondary.ncu-rep $P/secondary_r1.ncu-rep
  python tools/summarize_profiles.py --kernels $P/secondary_r1.ncu-rep > $P/SECONDARY_r1.txt
fi
[ -f gpurun_out/prof/timeline_c3.txt ] && grep -v Warn gpurun_out/prof/timeline_c3.txt | grep -v _warn_once > $P/timeline_c3_device.txt
[ -f gpurun_out/prof/timeline_c3_host.txt ] && grep -v Warn gpurun_out/prof/timeline_c3_host.txt | grep -v _warn_once > $P/timeline_c3_e2e.txt
[ -f gpurun_out/prof/io_bench.json ] && cp gpurun_out/prof/io_bench.json $P/io_bench_r1.json
[ -f gpurun_out/prof/pytest_gpu.log ] && tail -3 gpurun_out/prof/pytest_gpu.log > $P/pytest_gpu_r1.txt
[ -f gpurun_out/prof/gpu_check.log ] && cut -c1-600 gpurun_out/prof/gpu_check.log > $P/gpu_check_r1.txt
python tools/summarize_profiles.py --json $P/vote_banded_r1.ncu-rep | sed "s#\"source\": \"vote_banded_r1.ncu-rep\"#\"source\": \"$P/vote_banded_r1.ncu-rep\"#" > $P/vote_kernel_ncu.json
{ echo "# Round 1 measurement bundle (tools/profile_round.sh on one B200; see DESIGN.md section 6)"
  echo "# launch list = ncu of 'python bench.py --steps 2 --warmup 3 --no-cpu' (device solves AND pipelined e2e"
  echo "# solves, whose vote runs in 4 chunks: per-launch averages mix both; shares are what matter)"
  python tools/summarize_profiles.py $P/launches_r1.csv $P/vote_banded_r1.ncu-rep; } > $P/SUMMARY_r1.txt
echo refreshed
