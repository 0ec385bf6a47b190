for v in orig q; do cp _variants/$v.so paper_2502_06337_b200/_lib/librotavote_b200.so
ncu --set full --clock-control none -k regex:vote_banded -s 2 -c 1 -f -o gpurun_out/vote_$v python tools/profile_vote.py c3 3 > gpurun_out/ncu_$v.log 2>&1; echo $v rc=$?
done
cp _variants/q.so paper_2502_06337_b200/_lib/librotavote_b200.so
