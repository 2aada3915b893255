cd $GRAFT_REPO_ROOT
SEQCDC_WALKERS_PER_SM=1 python tools/tune.py markov 2 64 4 1 3 > gpurun_out/plain_lone.log 2>&1 &&
SEQCDC_WALKERS_PER_SM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 6 -c 1 -o gpurun_out/prof_lone2 -f python tools/tune.py markov 2 64 4 1 3 > gpurun_out/ncu_lone2.log 2>&1
echo "exit $?" >> gpurun_out/ncu_lone2.log
