"""Config-1 end-to-end step through the host C ABI, pipelined across steps.

One host thread issues the upload-heavy calls (compress A, compress B) and the
small record operations (scale, add, sub) of step k+1 while a second one issues
step k's three decompressions (downloads); the compressed records are
double-buffered by step parity.  Prints ms per step for the single-step op graph (bench.py's
`e2e`) and for the pipelined stream of steps.

    python tools/e2e_pipeline_probe.py [--steps 8]
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_13007_b200 as blz  # noqa: E402
from paper_2202_13007_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--timeline", action="store_true", help="print per-call start / end times of the pipelined run")
    ap.add_argument("--late-s", action="store_true", help="signal the sum's decompression after sub, not after add")
    ap.add_argument("--pageable", action="store_true", help="plain (pageable) host buffers instead of pinned ones")
    a = ap.parse_args()
    rows = cols = a.rows
    nbr, nbc = rows // 8, cols // 8
    nb = nbr * nbc
    hA = torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)
    hB = torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)
    hA.copy_(W.make("quadratic", rows, cols, seed=1, device="cuda"))
    hB.copy_(W.make("quadratic", rows, cols, seed=2, device="cuda"))
    npA, npB = hA.numpy(), hB.numpy()
    if a.pageable:
        import numpy as np
        npA, npB = np.array(npA), np.array(npB)

    def pinned_blocks():
        if a.pageable:
            import numpy as np
            return np.zeros(nb, blz.BLOCK_DTYPE)
        return torch.empty(nb * 48, dtype=torch.uint8, pin_memory=True).numpy().view(blz.BLOCK_DTYPE)

    def dense_out():
        if a.pageable:
            import numpy as np
            return np.empty((rows, cols), np.float64)
        return torch.empty((rows, cols), dtype=torch.float64, pin_memory=True).numpy()

    recs = [[pinned_blocks() for _ in range(5)] for _ in range(2)]  # cA cB cS cD cK per parity
    dout = dense_out()
    dout2 = dense_out()
    cx, cy, cz = blz.Context(0), blz.Context(0), blz.Context(0)
    lib = cx.lib
    P = lambda v: v.ctypes.data  # noqa: E731

    log = []

    def timed(who, name, k, fn):
        s0 = time.perf_counter()
        fn()
        log.append((who, name, k, s0, time.perf_counter()))

    def upload_side(ctx, k):
        """compress A, scale, compress B, add, sub (uploads and small record ops);
        yields after each result the other side consumes"""
        cA, cB, cS, cD, cK = recs[k % 2]
        h = ctx.handle
        timed("producer", "compress A", k, lambda: ctx.check(lib.blz_compress_matrix(h, P(npA), rows, cols, P(cA), 0)))
        timed("producer", "scale", k, lambda: ctx.check(lib.blz_mat_scale(h, P(cA), rows, cols, 3.5, P(cK), 0)))
        yield "k"
        timed("producer", "compress B", k, lambda: ctx.check(lib.blz_compress_matrix(h, P(npB), rows, cols, P(cB), 0)))
        timed("producer", "add", k,
              lambda: ctx.check(lib.blz_mat_add(h, P(cA), rows, cols, P(cB), rows, cols, P(cS), 0)))
        if not a.late_s:
            yield "s"
        timed("producer", "sub", k,
              lambda: ctx.check(lib.blz_mat_sub(h, P(cA), rows, cols, P(cB), rows, cols, P(cD), 0)))
        if a.late_s:  # the sum's decompression starts once sub is done: sub's small D2H
            yield "s"  # does not queue behind a 2 GiB download on the copy engine
        yield "d"

    def download_side(ctx, k, wait, tags=("k", "s", "d"), out=None):
        """decompressions (downloads) of the listed results"""
        cA, cB, cS, cD, cK = recs[k % 2]
        src = {"k": cK, "s": cS, "d": cD}
        for tag in tags:
            w0 = time.perf_counter()
            wait(tag)
            log.append(("consumer", "wait " + tag, k, w0, time.perf_counter()))
            timed("consumer", "decompress " + tag, k, lambda: ctx.check(
                lib.blz_decompress_matrix(ctx.handle, P(src[tag]), rows, cols, P(dout if out is None else out), 0)))

    def run_pipelined(n, two=False):
        ev = {(k, s): threading.Event() for k in range(n) for s in ("k", "s", "d", "done", "done2")}
        err = []

        def guard(fn):
            def run():
                try:
                    fn()
                except Exception as ex:  # noqa: BLE001
                    err.append(ex)
                    for e in ev.values():
                        e.set()
            return run

        def producer():
            for k in range(n):
                if k >= 2:  # records of parity k % 2 are free again
                    ev[(k - 2, "done")].wait()
                    if two:
                        ev[(k - 2, "done2")].wait()
                for tag in upload_side(cx, k):
                    ev[(k, tag)].set()

        def second():  # the add result's decompression on its own thread
            for k in range(n):
                download_side(cz, k, lambda tag, k=k: ev[(k, tag)].wait(), ("s",), dout2)
                ev[(k, "done2")].set()

        ths = [threading.Thread(target=guard(producer))] + ([threading.Thread(target=guard(second))] if two else [])
        for th in ths:
            th.start()
        for k in range(n):
            download_side(cy, k, lambda tag, k=k: ev[(k, tag)].wait(), ("k", "d") if two else ("k", "s", "d"))
            ev[(k, "done")].set()
        for th in ths:
            th.join()
        if err:
            raise err[0]

    def run_serial(n):
        for k in range(n):
            for _ in upload_side(cx, k):
                pass
            download_side(cx, k, lambda tag: None)

    run_serial(1)
    run_pipelined(2)
    torch.cuda.synchronize()
    run_pipelined(2, True)
    for name, fn in (("sequential", run_serial), ("pipelined", run_pipelined),
                     ("pipelined, two download threads", lambda n: run_pipelined(n, True))):
        t0 = time.perf_counter()
        fn(a.steps)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / a.steps
        print(f"{name}: {dt * 1e3:.1f} ms per step ({nb / dt / 1e6:.1f} M blocks/s) over {a.steps} steps", flush=True)
    if a.timeline:
        log.clear()
        t0 = time.perf_counter()
        run_pipelined(a.steps)
        torch.cuda.synchronize()
        for who, name, k, s0, s1 in sorted(log, key=lambda e: e[3]):
            print(f"{who:9s} step {k} {name:12s} {1e3 * (s0 - t0):8.1f} -> {1e3 * (s1 - t0):8.1f} ms ({1e3 * (s1 - s0):6.1f})")
    cx.close()
    cy.close()
    cz.close()


if __name__ == "__main__":
    main()
