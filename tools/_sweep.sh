cd $GRAFT_REPO_ROOT
for occ in 6 8 12 16 24; do
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py uniform 1 4096 16 0 10 >> gpurun_out/sweep21.jsonl 2>&1
  SEQCDC_WALKERS_PER_SM=$occ python tools/tune.py markov 2 4096 16 1 10 >> gpurun_out/sweep21.jsonl 2>&1
done
for fl in 32 64 128 256; do
  SEQCDC_G_FLOOR_CHUNKS=$fl python tools/tune.py uniform 1 4096 16 0 10 >> gpurun_out/sweep21.jsonl 2>&1
done
