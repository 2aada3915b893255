#!/bin/bash
# One GPU round trip: GPU parity tests, a bench line, the ncu launch list and
# one full ncu capture of the hot kernel.  Run under gpurun from the repo root.
#   tools/gpu_check.sh [tests|bench|ncu]...   (default: all three)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
steps="${*:-tests bench ncu}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt
for s in $steps; do
  case $s in
    tests)
      timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
      echo "pytest -m gpu exit $?" >> gpurun_out/summary.txt ;;
    bench)
      timeout 400 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1
      echo "bench exit $?" >> gpurun_out/summary.txt ;;
    ncu)
      timeout 400 python bench.py --steps 3 --warmup 3 > gpurun_out/plain.log 2>&1 &&
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1 &&
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 4 -c 1 \
          -o gpurun_out/prof_walk -f python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_full.log 2>&1
      echo "ncu exit $?" >> gpurun_out/summary.txt ;;
  esac
done
cat gpurun_out/summary.txt
