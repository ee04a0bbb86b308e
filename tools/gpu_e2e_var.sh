for i in 1 2 3; do
HSDE_TIMING=1 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu > gpurun_out/e2ev_$i.json 2> gpurun_out/e2ev_$i.err
python - <<PY
import json,re
b=json.loads(open('gpurun_out/e2ev_$i.json').read())
print($i, b['e2e']['walls_s'])
big=[l.strip() for l in open('gpurun_out/e2ev_$i.err') if re.search(r'(\d+\.\d) ms', l) and float(re.search(r'(\d+\.\d) ms', l).group(1))>30]
print(big)
PY
done
