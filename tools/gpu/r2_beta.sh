set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_beta.py -m gpu -q -s 2>&1 | grep -E 'beta |passed|failed|Error|assert' | tail -30
rm -f gpurun_out/sanitize2.txt
for tool in racecheck synccheck; do
  echo "== $tool" >> gpurun_out/sanitize2.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py >> gpurun_out/sanitize2.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize2.txt
done
grep -E '^==|SUMMARY|rc=|sanitize_small|Warning|hazard' gpurun_out/sanitize2.txt | head -40
