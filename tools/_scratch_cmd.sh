#!/bin/bash
# evidence refresh at HEAD (GPU box): GPU suite, smoke, bench line, launch list,
# ncu captures, per-kernel roofline, every-ray parity table
tag=${1:-r2h}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${tag}.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_${tag}.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench_${tag}.err
cp gpurun_out/bench.json gpurun_out/bench_${tag}.json
RSI_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-configs \
  > gpurun_out/torchrun_w2_${tag}.json 2> gpurun_out/torchrun_w2_${tag}.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err
bash tools/profile.sh ${tag} > /dev/null 2>&1
bash tools/kernel_roofline.sh ${tag} > /dev/null 2>&1
timeout 900 python tools/parity_report.py > gpurun_out/parity_${tag}.txt 2> gpurun_out/parity_${tag}.err
tail -3 gpurun_out/pytest_gpu_${tag}.log
