"""C4 (CFG=C3: C3) block sweeps under sustained load with the SM clock and throttle
reasons sampled (bench.ClockSampler), for GPSPCA_TC_PROBE power experiments
(probe 1024: T1 issues one MMA per TMEM segment instead of one per 16 rows --
results wrong by design)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_1312_6182_b200 as gps
    from paper_1312_6182_b200 import _native
    from paper_1312_6182_b200.block import BlockLoop, _top_m_columns

    want = os.environ.get("CFG", "C4")
    name, p, n, m, pen, mu, frac, data, k = [c for c in bench.BLOCK_CONFIGS if c[0] == want][0]
    dev = torch.device("cuda", 0)
    n_classes, n_factors, support = (16, 10, n // 200) if name == "C3" else (32, 64, n // 128)
    At = bench.make_lowrank(torch, p, n, 0, n, dev, n_classes, n_factors, support)
    A = gps.DataMatrix.from_device(At.data_ptr(), p, n, owner=At, device=0)
    top = frac * float(A.norms.max())
    iters = int(os.environ.get("ITERS", 40))
    loop = BlockLoop(A, pen, m, np.full(m, top if pen == "l1" else top * top), mu, 0.0, iters + 8)
    loop.start_columns(_top_m_columns(np.asarray(A.norms), m))
    L = _native.lib()
    s = torch.cuda.Stream(dev)
    A.context.set_stream(s.cuda_stream)
    # sweeps only (T0, T1, T1x, T1s, T2, K2): the probe's wrong results must
    # not stop the loop through the polar step
    for _ in range(3):
        _native.check(L.gps_bk_enqueue_sweep(loop.handle))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(0) as clocks:
        e0.record(s)
        for _ in range(iters):
            _native.check(L.gps_bk_enqueue_sweep(loop.handle))
        e1.record(s)
        e1.synchronize()
    A.context.set_stream(None)
    d, it, _ = bench._bk_poll(loop)
    print(f"probe={os.environ.get('GPSPCA_TC_PROBE', '0')} {name} sweep {e0.elapsed_time(e1) / iters:.3f} ms "
          f"clocks {clocks.summary()} (loop done={d} at iteration {it})", flush=True)


if __name__ == "__main__":
    main()
