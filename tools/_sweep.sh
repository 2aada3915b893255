cd $GRAFT_REPO_ROOT
tools/gpu_check.sh tests
for occ in 16 24; do
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py markov 2 1024 4 1 >> gpurun_out/sweep6.jsonl 2>&1
done
SEQCDC_WALKERS_PER_SM=12 python tools/tune.py uniform 1 1024 8 0 >> gpurun_out/sweep6.jsonl 2>&1
SEQCDC_WALKERS_PER_SM=8 python tools/tune.py uniform 1 1024 16 0 >> gpurun_out/sweep6.jsonl 2>&1
python tools/tune.py markov 2 4096 4 1 >> gpurun_out/sweep6.jsonl 2>&1
python tools/tune.py rampmix 5 4096 8 0 >> gpurun_out/sweep6.jsonl 2>&1
python tools/tune.py uniform 1 4096 16 0 >> gpurun_out/sweep6.jsonl 2>&1
