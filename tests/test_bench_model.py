"""CPU checks of bench.py's roofline model against SURVEY.md §8(d) and of the
DDP hook's host logic (no GPU)."""

import pytest

import bench
from paper_2310_06993_b200.ddp_hook import OptiReduceState, max_bucket_len_for


@pytest.mark.parametrize("n,L,hbm_mb,nvl_mb", [
    (8, 25_000_000, 619.4, 234.9),      # headline, N=8
    (4, 25_000_000, 636.2, 201.3),      # headline, N=4
    (2, 25_000_000, 669.8, 134.2),      # headline, N=2
    (8, 6_553_600, 157.3, 58.7),        # 25 MB bucket, RHT on
])
def test_step_alg_bytes_match_survey(n, L, hbm_mb, nvl_mb):
    hbm, nvl = bench.step_alg_bytes([L], n, 4, 4, True)
    assert abs(hbm / 1e6 - hbm_mb) < 0.1
    assert abs(nvl / 1e6 - nvl_mb) < 0.1


def test_step_alg_bytes_rht_off_and_bf16():
    # RHT off, 25 MB bucket, N=8 (SURVEY: 81.9 MB HBM, 45.9 MB NVLink)
    hbm, nvl = bench.step_alg_bytes([6_553_600], 8, 4, 4, False)
    assert abs(hbm / 1e6 - 81.9) < 0.1 and abs(nvl / 1e6 - 45.9) < 0.1
    # GPT-2 XL bf16 buckets (bf16 in and out, fp32 aggregate), 2^24 (SURVEY: 262.1 MB, 117.4 MB)
    hbm, nvl = bench.step_alg_bytes([13_107_200], 8, 2, 2, True)
    assert abs(hbm / 1e6 - 262.1) < 0.1 and abs(nvl / 1e6 - 117.4) < 0.1


def test_kernel_bytes_classes():
    dim, L, n = 1 << 23, 6_553_600, 4
    for cls in ("enc_first", "enc_last", "enc_mean", "aggregate", "dec_first", "dec_last", "fused", "prep", "small"):
        assert bench.kernel_bytes(cls, dim, L, n, 4, 4) > 0
    # the fused last-pass + stage-1 mean reads the wire once and writes one
    # shard's mean per worker: less than the last pass plus the aggregate
    assert bench.kernel_bytes("enc_mean", dim, L, n, 4, 4) < (bench.kernel_bytes("enc_last", dim, L, n, 4, 4)
                                                               + bench.kernel_bytes("aggregate", dim, L, n, 4, 4))


def test_ddp_hook_host_logic():
    torch = pytest.importorskip("torch")
    model = torch.nn.Sequential(torch.nn.Linear(100, 50), torch.nn.Linear(50, 7))
    cap = int(1.0 * 1024 * 1024 // 4)
    assert max_bucket_len_for(model, 1.0) == cap + 100 * 50 + 1024
    st = OptiReduceState(drop_prob=0.0)
    assert st.masks(3).kind == "none"
    st = OptiReduceState(drop_prob=0.02, seed=5)
    a, b = st.masks(1), st.masks(1)
    assert a.kind == "coin" and a.seed == b.seed and a.drop_prob == 0.02
    st.generation += 1
    assert st.masks(1).seed != a.seed  # per generation (and bucket) coin streams
    assert st.masks(2).seed != st.masks(1).seed


def test_reference_arm_json_contract():
    """`bench.py --impl reference` (the driver's reference arm: the oracle port
    on the host cores, no GPU) prints one JSON line with the contract's keys,
    on our arm's metric / unit / config."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1", "--steps", "1",
                          "--warmup", "1"], cwd=root, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [line for line in res.stdout.splitlines() if line.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"] == "bucket allreduce GB/s (TAR+RHT)" and d["unit"] == "GB/s"
    assert d["config"]["workload"] == "cfg1" and d["config"]["same_config"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
