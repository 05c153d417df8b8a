#!/bin/bash
# BASELINE configs: sweep (1 GPU and all GPUs), BERT RHT on/off, GPT-2 XL bf16, cfg1, tests
OUT=gpurun_out/$1; mkdir -p $OUT
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc $?" >> $OUT/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/sweep.py --workers 4 > $OUT/sweep_1gpu.jsonl 2> $OUT/sweep_1gpu.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 tools/sweep.py > $OUT/sweep_n$N.jsonl 2> $OUT/sweep_n$N.err
for HT in on off; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29535 \
    bench.py --gpus $N --steps 3 --warmup 3 --workload bert --ht $HT > $OUT/bench_bert_ht${HT}_n$N.log 2>&1
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29536 \
    bench.py --gpus $N --steps 3 --warmup 3 --workload gpt2xl --drop 0.05 > $OUT/bench_gpt2xl_n$N.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --workload cfg1 > $OUT/bench_cfg1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --drop 0 > $OUT/bench_resnet_drop0.log 2>&1
echo done
