cd $GRAFT_REPO_ROOT
SEQCDC_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --bytes-per-gpu 536870912 > gpurun_out/bench_n2_gloo.log 2>&1
echo "exit $?" >> gpurun_out/bench_n2_gloo.log
