# Final verification of the committed state: GPU suite, smoke, bench line.
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/s3_verify_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s3_verify_bench.json 2> gpurun_out/s3_verify_bench.err; python -c "
import json; d=json.loads([l for l in open('gpurun_out/s3_verify_bench.json') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
