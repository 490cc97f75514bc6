mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/san/san_$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/san/summary.txt
done
timeout 600 python tools/run_reference_tests.py -q > gpurun_out/san/reference_suite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/san/summary.txt
