echo "== synccheck serial" > gpurun_out/sync3.txt
GLA_SERIAL=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 3 python tools/sanitize_small.py >> gpurun_out/sync3.txt 2>&1
echo "== racecheck warn detail" >> gpurun_out/sync3.txt
timeout 900 compute-sanitizer --tool racecheck --print-level info --print-limit 5 python tools/sanitize_small.py >> gpurun_out/sync3.txt 2>&1
timeout 600 python -m pytest tests/test_layer.py -m gpu -q -s 2>&1 | tail -8 >> gpurun_out/sync3.txt
