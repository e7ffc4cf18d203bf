t0=$(date +%s); timeout 600 python bench.py > gpurun_out/s3_bench2.json 2> gpurun_out/s3_bench2.err; t1=$(date +%s); echo "bench wall $((t1 - t0)) s"
python -c "
import json; d=json.loads([l for l in open('gpurun_out/s3_bench2.json') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['cpu_baseline'])"
