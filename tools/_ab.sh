# A/B of library variants (tuning only): tools/_ab.sh VARIANT...
for v in "$@"; do
  echo "== lib $v"
  SEQCDC_LIB=$v python tools/lone.py 1024 16
  for i in 1 2; do SEQCDC_LIB=$v python tools/tune.py markov 1 1024 4 1 20; done
  SEQCDC_LIB=$v python tools/tune.py markov 1 4096 4 1 10
  SEQCDC_LIB=$v python tools/tune.py rampmix 1 4096 8 0 10
  SEQCDC_LIB=$v python tools/tune.py uniform 1 4096 16 0 10
done
