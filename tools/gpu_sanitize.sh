# compute-sanitizer memcheck / racecheck / synccheck over small launches of every kernel family
# (tools/sanitize_small.py) -> gpurun_out/san/
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_small.py > gpurun_out/san/san_$t.log 2>&1
done
