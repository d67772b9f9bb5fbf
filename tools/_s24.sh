O=gpurun_out/s24; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_all.log 2>&1; echo "exit $?" >> $O/pytest_gpu_all.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
echo done > $O/DONE
