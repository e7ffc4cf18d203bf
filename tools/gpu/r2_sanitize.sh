mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/sanitize.txt
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py >> gpurun_out/sanitize.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize.txt
done
