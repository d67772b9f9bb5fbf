#!/bin/bash
# One gpurun session: GPU parity tests, bench per compositor variant, launch list, ncu --set full captures.
#   gpurun --timeout 2400 -- 'bash tools/gpu_session.sh <tag>'
# env: VARIANTS="mp direct" (GB_COMPOSITOR values benched), ALT_TESTS="direct" (variants parity-tested on a
#      subset besides the default), NCU=1 (launch list + full K3/K4 captures of the default variant),
#      REF=1 (bench --impl reference), TESTS=1 (full -m gpu suite)
# Everything lands in gpurun_out/<tag>/.
TAG=${1:-s}
O=gpurun_out/$TAG
mkdir -p $O
VARIANTS=${VARIANTS:-direct}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  if [ "${FULL:-0}" = 1 ]; then K=""; else K="not configs2_full"; fi
  timeout 2400 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
  echo "smoke exit $?" >> $O/smoke.log
fi
# variant names: direct (default), staged, grp (G=8), grp16/grp4, backward-only grp (grp16b, grp16bu, grp8b),
# fused (gb_render_loss_backward), nofuse, blocking (blocking binning), eager (no CUDA graph), lanes2
venv() { case $1 in grp16) echo "GB_COMPOSITOR=grp GB_GROUP=16";; grp4) echo "GB_COMPOSITOR=grp GB_GROUP=4";; grp16b) echo "GB_COMPOSITOR_BWD=grp GB_GROUP=16";; grp16bu) echo "GB_COMPOSITOR_BWD=grp GB_GROUP=16 GB_GRP_TEXEL=uni";; grp8b) echo "GB_COMPOSITOR_BWD=grp GB_GROUP=8";; nofuse) echo "GB_NO_FUSE=1";; fused) echo "GB_FUSED=1";; blocking) echo "GB_BLOCKING_BINNING=1";; eager) echo "GB_GRAPH=0";; lanes2) echo "GB_LANES=2";; *) echo "GB_COMPOSITOR=$1";; esac; }
for v in ${ALT_TESTS:-}; do
  env $(venv $v) timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "configs1 or pinhole_small or ortho_random or ragged" > $O/pytest_gpu_$v.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu_$v.log
done
for v in $VARIANTS; do
  env $(venv $v) timeout 600 python bench.py --no-cpu-baseline > $O/bench_$v.json 2> $O/bench_$v.err
  echo "bench exit $?" >> $O/bench_$v.err
done
if [ "${DBG:-0}" = 1 ]; then
  GB_COMPOSITOR=direct timeout 600 python tools/dbg_run.py > $O/dbg_counters.txt 2>&1
fi
if [ "${SWEEP:-0}" = 1 ]; then
  timeout 1200 python tools/sweep.py --out $O/sweep > $O/sweep.log 2>&1
fi
if [ "${REF:-0}" = 1 ]; then
  timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
  timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err
fi
if [ "${NCU:-1}" = 1 ]; then
  env $(venv ${NCU_VARIANT:-direct}) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
  env $(venv ${NCU_VARIANT:-direct}) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_backward -s 8 -c 1 \
    -o $O/k4_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k4.log 2>&1
  env $(venv ${NCU_VARIANT:-direct}) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 8 -c 1 \
    -o $O/k3_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k3.log 2>&1
  env $(venv ${NCU_VARIANT:-direct}) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 8 -c 1 \
    -o $O/kf_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_kf.log 2>&1
fi
echo done > $O/DONE
