for v in tl5 tl5m5 tl5m4 tl4m4; do RSI_LIB=paper_2305_01867_b200/lib/librsi_$v.so timeout 300 python bench.py --no-configs --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2>&1; done
