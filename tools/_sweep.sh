cd $GRAFT_REPO_ROOT
SEQCDC_LIB=build/v_sp.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -m gpu -q -x > gpurun_out/pytest_sp.log 2>&1
for v in v24 sp sph2 sph4; do
  export SEQCDC_LIB=build/v_$v.so
  python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep19.jsonl 2>&1
  python tools/tune.py rampmix 5 4096 8 0 10 >> gpurun_out/sweep19.jsonl 2>&1
  python tools/tune.py uniform 1 4096 16 0 10 >> gpurun_out/sweep19.jsonl 2>&1
  python tools/tune.py uniform 1 4096 8 0 10 >> gpurun_out/sweep19.jsonl 2>&1
  python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep19.jsonl 2>&1
done
