#!/bin/bash
# One gpurun session: GPU parity tests, bench (both K3/K4 variants), launch list, one ncu --set full capture.
#   gpurun --timeout 2400 -- 'bash tools/gpu_session.sh [tag]'
# Everything lands in gpurun_out/<tag>/.
TAG=${1:-s}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "not configs2_full" > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench exit $?" >> $O/bench.err
GB_TUNE_DIRECT=3 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_direct.json 2> $O/bench_direct.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
# launch list (cold-cache, serialised; share of step only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
# one full capture of the dominant kernel (K4) and K3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_backward -s 8 -c 1 \
  -o $O/k4_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 8 -c 1 \
  -o $O/k3_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k3.log 2>&1
echo done > $O/DONE
