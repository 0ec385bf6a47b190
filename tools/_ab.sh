for v in red2 red4 red8 red2 red4 red8; do cp _variants/$v.so paper_2502_06337_b200/_lib/librotavote_b200.so
python tools/timeline.py c3 > gpurun_out/tl_dev.txt 2>&1
python tools/timeline.py c3 host > gpurun_out/tl_host.txt 2>&1
echo $v $(grep reduce gpurun_out/tl_dev.txt | awk '{print $4}') $(grep reduce gpurun_out/tl_host.txt | awk '{print $4}') $(grep span gpurun_out/tl_dev.txt gpurun_out/tl_host.txt | awk '{print $2}')
done
