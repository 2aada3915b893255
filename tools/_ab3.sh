# walkers-per-SM on 1 GiB Markov 4K, several seeds (tuning only)
for s in 1 2 3 4 5 6; do
  for w in 21 22 23; do
    SEQCDC_WALKERS_PER_SM=$w python tools/tune.py markov $s 1024 4 1 20
  done
done
