O=gpurun_out/s26; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_all.log 2>&1; echo "exit $?" >> $O/pytest_gpu_all.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 8 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
echo done > $O/DONE
