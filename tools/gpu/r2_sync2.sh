echo "== synccheck GLA_DQ3=1" > gpurun_out/sync2.txt
GLA_DQ3=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 3 python tools/sanitize_small.py >> gpurun_out/sync2.txt 2>&1
echo "== racecheck (hazard detail)" >> gpurun_out/sync2.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 python tools/sanitize_small.py >> gpurun_out/sync2.txt 2>&1
