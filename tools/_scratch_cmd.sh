python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "overflow or launch_counter or stacked or terrain or sphere_all or dedup or fuzz or chain" > gpurun_out/pt_b.log 2>&1
echo "exit $?" >> gpurun_out/pt_b.log
timeout 600 python bench.py --mode intercept_count --no-configs --no-cpu-baseline --no-e2e --no-extra-modes > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv python bench.py --mode intercept_count --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-e2e --no-extra-modes > /dev/null 2>&1
tail -3 gpurun_out/pt_b.log
