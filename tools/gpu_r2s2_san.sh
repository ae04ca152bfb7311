for tool in memcheck synccheck; do timeout 1500 compute-sanitizer --tool $tool python tools/sanitize.py > gpurun_out/san_$tool.txt 2>&1; tail -3 gpurun_out/san_$tool.txt; done
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize.py > gpurun_out/san_racecheck.txt 2>&1; tail -3 gpurun_out/san_racecheck.txt
