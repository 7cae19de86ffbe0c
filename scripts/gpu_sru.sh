for r in 1 2; do for u in 5 6 7 8; do
  LPQ_SR_U=$u timeout 300 python bench.py --config c1 --no-cpu > gpurun_out/sru.$u.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/sru.$u.json')); print('u=$u c1', d['value'])"
  LPQ_SR_U=$u timeout 300 python bench.py --config c1log --no-cpu > gpurun_out/sru.$u.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/sru.$u.json')); print('u=$u c1log', d['value'])"
done; done
