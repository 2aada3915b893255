cd $GRAFT_REPO_ROOT
python tools/tune.py markov 2 1024 4 1 3 > gpurun_out/plain_post.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stitch|k_copy" -s 6 -c 2 -o gpurun_out/prof_post -f python tools/tune.py markov 2 1024 4 1 3 > gpurun_out/ncu_post.log 2>&1
echo "exit $?" >> gpurun_out/ncu_post.log
