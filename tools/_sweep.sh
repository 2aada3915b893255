cd $GRAFT_REPO_ROOT
for spw in 100 125 150 200 300; do
  SEQCDC_G_FLOOR_CHUNKS=2 SEQCDC_SEGS_PER_WALKER_X100=$spw python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep16.jsonl 2>&1
done
for spw in 100 150 200; do
  SEQCDC_G_FLOOR_CHUNKS=2 SEQCDC_SEGS_PER_WALKER_X100=$spw python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep16.jsonl 2>&1
done
