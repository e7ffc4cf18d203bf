# Full GPU test suite, smoke, then compute-sanitizer (memcheck / racecheck / synccheck) on small shapes.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 | tee gpurun_out/r2_gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
rm -f gpurun_out/sanitize.txt
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/sanitize.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py >> gpurun_out/sanitize.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize.txt
done
grep -E '^==|ERROR SUMMARY|rc=|sanitize_small' gpurun_out/sanitize.txt
