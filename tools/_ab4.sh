# dynamic (warp-slot sized) layout vs static, several seeds (tuning only)
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for s in 1 2 3 4; do
  for d in 0 1; do SEQCDC_DYN=$d python tools/tune.py markov $s 1024 4 1 20; done
done
for d in 0 1; do SEQCDC_DYN=$d python tools/tune.py markov 1 4096 4 1 10; SEQCDC_DYN=$d python tools/tune.py rampmix 1 4096 8 0 10; SEQCDC_DYN=$d python tools/tune.py uniform 1 4096 16 0 10; done
