cd $GRAFT_REPO_ROOT
for v in v24 b2n4 b512; do
  export SEQCDC_LIB=build/v_$v.so
  python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep10.jsonl 2>&1
  SEQCDC_WALKERS_PER_SM=22 python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep10.jsonl 2>&1
  SEQCDC_WALKERS_PER_SM=2 python tools/tune.py markov 2 1024 4 1 5 >> gpurun_out/sweep10.jsonl 2>&1
  python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep10.jsonl 2>&1
  SEQCDC_WALKERS_PER_SM=12 python tools/tune.py uniform 1 1024 8 0 >> gpurun_out/sweep10.jsonl 2>&1
done
