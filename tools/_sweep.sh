cd $GRAFT_REPO_ROOT
for occ in 19 20 21 22 23 24; do
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py markov 2 1024 4 1 30 >> gpurun_out/sweep18.jsonl 2>&1
done
for occ in 20 22 24; do
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep18.jsonl 2>&1
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py rampmix 5 4096 8 0 10 >> gpurun_out/sweep18.jsonl 2>&1
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py markov 7 2048 4 1 10 >> gpurun_out/sweep18.jsonl 2>&1
done
