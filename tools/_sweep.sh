cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -m gpu -q -x > gpurun_out/pytest_quick.log 2>&1
for wgt in 0 1; do
  for i in 1 2; do SEQCDC_WEIGHTED=$wgt python tools/tune.py markov 2 1024 4 1 30 >> gpurun_out/sweep26.jsonl 2>&1; done
  SEQCDC_WEIGHTED=$wgt python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep26.jsonl 2>&1
  SEQCDC_WEIGHTED=$wgt python tools/tune.py rampmix 5 4096 8 0 10 >> gpurun_out/sweep26.jsonl 2>&1
  SEQCDC_WEIGHTED=$wgt python tools/tune.py uniform 1 4096 8 0 10 >> gpurun_out/sweep26.jsonl 2>&1
done
SEQCDC_LIB=build/v_tl.so TL_SAVE=gpurun_out/tl_w2.npy python tools/timeline.py markov 2 1024 4 1 > gpurun_out/tl26.jsonl 2>&1
