for AB in ${ABS:-0 4}; do
  OPTR_AB=$AB timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$AB bench.py --gpus 2 --steps 20 --workload headline --no-cpu-baseline > gpurun_out/ab3/h$AB.log 2>&1
  OPTR_AB=$AB timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$AB bench.py --gpus 2 --steps 20 --no-cpu-baseline > gpurun_out/ab3/r$AB.log 2>&1
done
