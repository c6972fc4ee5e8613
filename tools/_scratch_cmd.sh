for v in tl0; do RSI_LIB=paper_2305_01867_b200/lib/librsi_$v.so timeout 300 python bench.py --workload sphere1m --no-configs --no-cpu-baseline --no-e2e > gpurun_out/bench_1m_$v.json 2>&1; done
timeout 300 python bench.py --workload sphere1m --no-configs --no-cpu-baseline --no-e2e > gpurun_out/bench_1m_tl5.json 2>&1
