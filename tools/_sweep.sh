cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_quick.log 2>&1
python tools/tune.py markov 2 1024 4 1 20 >> gpurun_out/sweep20.jsonl 2>&1
python tools/tune.py zeroheavy 3 1024 4 0 10 >> gpurun_out/sweep20.jsonl 2>&1
python tools/tune.py zeroheavy 3 1024 8 0 10 >> gpurun_out/sweep20.jsonl 2>&1
python tools/configs_bench.py 3 >> gpurun_out/cfg3.jsonl 2>&1
