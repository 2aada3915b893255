cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_quick.log 2>&1
python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep14.jsonl 2>&1
SEQCDC_WALKERS_PER_SM=22 python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep14.jsonl 2>&1
SEQCDC_WALKERS_PER_SM=1 python tools/tune.py markov 2 64 4 1 5 >> gpurun_out/sweep14.jsonl 2>&1
python tools/tune.py markov 2 4096 4 1 10 >> gpurun_out/sweep14.jsonl 2>&1
SEQCDC_WALKERS_PER_SM=12 python tools/tune.py uniform 1 1024 8 0 >> gpurun_out/sweep14.jsonl 2>&1
