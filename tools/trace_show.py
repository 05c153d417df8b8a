"""Summarise fused-kernel traces written by tools/fused_trace.py."""
import sys

import numpy as np

tag = sys.argv[1]
for r in range(8):
    try:
        a = np.load(f"gpurun_out/{tag}/trace_r{r}.npy").astype(np.int64)
    except FileNotFoundError:
        continue
    cap = a.shape[1]
    ed = a[:, :cap // 2]
    ag = a[:, cap // 2:]
    ed = ed[ed[:, :, 3] != 0]
    ag = ag[ag[:, :, 3] != 0]
    t0 = min(ed[:, 1].min(), ag[:, 1].min() if len(ag) else 1 << 62)
    kind = ed[:, 0] >> 28
    print(f"== rank {r}: span {(max(ed[:, 3].max(), ag[:, 3].max()) - t0) / 1e3:.1f} us")
    for k, name in ((0, "E"), (2, "D")):
        m = kind == k
        if m.sum() == 0:
            continue
        wait = (ed[m, 2] - ed[m, 1]) / 1e3
        work = (ed[m, 3] - ed[m, 2]) / 1e3
        ends = (ed[m, 3] - t0) / 1e3
        print(f"  {name}: n={m.sum()} wait mean {wait.mean():.2f} max {wait.max():.1f} work mean {work.mean():.2f}"
              f" | end pct {np.round(np.percentile(ends, [0, 10, 50, 90, 100]), 1)}")
    if len(ag):
        cw = (ag[:, 2] - ag[:, 1]) / 1e3
        wk = (ag[:, 3] - ag[:, 2]) / 1e3
        pub = (ag[:, 3] - t0) / 1e3
        print(f"  A: n={len(ag)} claim->ready mean {cw.mean():.2f} max {cw.max():.1f}; ready->pub mean {wk.mean():.2f}"
              f" max {wk.max():.1f} | pub pct {np.round(np.percentile(pub, [0, 10, 50, 90, 100]), 1)}")
