cd $GRAFT_REPO_ROOT
for occ in 18 20 22 23 24 25; do
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep9.jsonl 2>&1
done
for occ in 20 24 25; do
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep9.jsonl 2>&1
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py rampmix 5 4096 8 0 10 >> gpurun_out/sweep9.jsonl 2>&1
done
