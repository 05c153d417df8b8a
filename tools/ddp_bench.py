"""DDP training-step benchmark: PyTorch DDP over NCCL with its default
all-reduce vs the OptiReduce comm hook (lossless RHT, 1% seeded drops, and a
capped fused-kernel grid), one process per GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/ddp_bench.py \
        [--model resnet50|gpt2] [--steps 20] [--warmup 5]

A step = forward + backward (the hook runs inside backward, overlapped with
it) + SGD update, bf16 autocast, synthetic data, random init.  Prints one
JSON line per mode (rank 0): ms per step (CUDA events, max over ranks).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def build(model_name, dev):
    if model_name == "resnet50":
        import torchvision

        model = torchvision.models.resnet50().to(dev)
        x = torch.randn(64, 3, 224, 224, device=dev)
        y = torch.randint(0, 1000, (64,), device=dev)

        def loss_fn(m):
            return torch.nn.functional.cross_entropy(m(x), y)
    else:
        from transformers import GPT2Config, GPT2LMHeadModel

        cfg = GPT2Config(n_positions=1024, n_embd=768, n_layer=12, n_head=12)
        model = GPT2LMHeadModel(cfg).to(dev)
        ids = torch.randint(0, cfg.vocab_size, (8, 1024), device=dev)

        def loss_fn(m):
            return m(input_ids=ids, labels=ids).loss
    return model, loss_fn


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50", choices=["resnet50", "gpt2"])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ctas", default="32", help="comma list of fused-kernel CTA caps to time as extra modes")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2310_06993_b200.ddp_hook import OptiReduceState, max_bucket_len_for, optireduce_hook

    modes = [("nccl_allreduce", None), ("noop_hook", None), ("optireduce_lossless", dict(drop_prob=0.0)),
             ("optireduce_1pct_drops", dict(drop_prob=0.01))]
    modes += [(f"optireduce_lossless_{c}ctas", dict(drop_prob=0.0, fused_ctas=int(c)))
              for c in args.ctas.split(",") if c]
    for name, hook_kw in modes:
        torch.manual_seed(0)
        model, loss_fn = build(args.model, dev)
        ddp = DDP(model, device_ids=[dev.index], bucket_cap_mb=25)
        state = None
        if name == "noop_hook":  # hook framework cost alone: no communication at all
            def noop(_st, bucket):
                fut = torch.futures.Future()
                fut.set_result(bucket.buffer())
                return fut
            ddp.register_comm_hook(None, noop)
            hook_kw = None
        elif hook_kw is not None:
            state = OptiReduceState(max_bucket_len=max_bucket_len_for(model, 25), ht=True, seed=1, **hook_kw)
            ddp.register_comm_hook(state, optireduce_hook)
        opt = torch.optim.SGD(ddp.parameters(), lr=1e-3)

        def step():
            opt.zero_grad(set_to_none=True)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = loss_fn(ddp)
            loss.backward()
            opt.step()

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nparams = sum(p.numel() for p in model.parameters())
        if rank == 0:
            print(json.dumps({"model": args.model, "mode": name, "gpus": world, "ms_per_step": round(t.item(), 3),
                              "params": nparams, "steps": args.steps, "bucket_cap_mb": 25,
                              "buckets_per_step": len(state.received) if state else None}), flush=True)
        if state is not None and state.comm is not None:
            state.comm.close()
        del ddp, model, opt
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
