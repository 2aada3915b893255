cd $GRAFT_REPO_ROOT
python tools/dedup_bench.py 2 > gpurun_out/plain_dd.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sha256 -s 2 -c 1 -o gpurun_out/prof_sha -f python tools/dedup_bench.py 2 > gpurun_out/ncu_sha.log 2>&1
echo "exit $?" >> gpurun_out/ncu_sha.log
