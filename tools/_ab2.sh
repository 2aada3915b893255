# walkers-per-SM x ring-geometry sweep (tuning only)
for v in build/v_base.so build/v_r4k.so build/v_r1k8.so; do
  for w in 22 24 26 28 32; do
    for args in "markov 1 1024 4 1 20" "markov 1 4096 4 1 10" "uniform 1 4096 4 0 10"; do
      SEQCDC_WALKERS_PER_SM=$w SEQCDC_LIB=$v python tools/tune.py $args
    done
  done
done
