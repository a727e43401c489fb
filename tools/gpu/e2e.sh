python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/e2e_2d.jsonl 2>gpurun_out/e2e_2d.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/e2e_2d.jsonl').read()); print('2d', d['value'], d['e2e'])"
