set -x
timeout 600 ncu --section WarpStateStats --section SourceCounters --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k regex:mlp_tc -s 9 -c 1 -o gpurun_out/tc_src python tools/kernel_bench.py 21 4 > gpurun_out/tc_src.log 2>&1
tail -2 gpurun_out/tc_src.log
