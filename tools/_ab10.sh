# batch segments-per-walker default check (tuning only)
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do
  python tools/configs_bench.py 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'config' in d: print('cfg3', d['workload'][-16:], d['GBps'], d['bit_exact'])"
done
