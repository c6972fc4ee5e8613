for v in base nopt c32 hint1; do
RSI_LIB=paper_2305_01867_b200/lib/librsi_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sphere or terrain or vertices or stacked or single or fuzz or compaction or sparse or bench_size" 2>&1 | tail -1 | sed "s/^/[$v parity] /"
for wl in sphere paper_terrain; do
RSI_LIB=paper_2305_01867_b200/lib/librsi_$v.so WL=$wl timeout 300 python tools/sweep.py 2>&1 | grep "bary.*ms" | sed "s/^/[$v $wl] /"
done
RSI_LIB=paper_2305_01867_b200/lib/librsi_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_trace -c 1 --csv --log-file gpurun_out/dram_$v.csv python bench.py --mode barycentric --steps 1 --warmup 3 --no-configs --no-cpu-baseline --no-e2e --no-extra-modes --rays-per-gpu 10000000 > /dev/null 2>&1
done
