# decision variants (tuning only): default (REDUX bulk for single streams, ballots for batches) vs forced
for v in "" build/v_allred.so build/v_allbal.so ""; do
  echo "== ${v:-default}"
  SEQCDC_LIB=$v python tools/configs_bench.py 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'config' in d: print('cfg3', d['workload'][-16:], d['GBps'])"
  for args in "markov 2 1024 4 1 20" "markov 1 4096 4 1 10"; do
    SEQCDC_LIB=$v python tools/tune.py $args | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['kind'], d['MiB'], d['GBps'], d['walk_GBps'])"; done
done
