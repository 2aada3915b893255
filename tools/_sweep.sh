cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_range.py -m gpu -q -x > gpurun_out/pytest_quick.log 2>&1
for i in 1 2; do python tools/tune.py markov 2 1024 4 1 30 >> gpurun_out/sweep22.jsonl 2>&1; done
SEQCDC_WALKERS_PER_SM=1 python tools/tune.py markov 2 64 4 1 5 >> gpurun_out/sweep22.jsonl 2>&1
python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep22.jsonl 2>&1
