"""Handles in several host threads (the header: a handle is not thread-safe, one per host thread):
the library's process-wide state -- the run-time NCCL loader, the TMA encoder entry point, the
TF32 tile-list cache -- is shared under a lock, so concurrent calls on separate handles and
streams give the same results as sequential ones (fp64: bitwise; the path is deterministic)."""

import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def test_concurrent_handles_match_sequential():
    import torch
    import paper_1705_07112_b200 as P
    kern = {"kind": "soft", "tau": 0.2, "tau_relative": True}
    Xs = [torch.from_numpy(W.random_dense(300 + 37 * i, 500, seed=i)).cuda() for i in range(4)]
    X32 = [x.float() for x in Xs]
    # sequential references
    h0 = P.Handle(0)
    ref64 = [h0.apply(x, kern, 12, T=40).cpu() for x in Xs]
    ref32 = [h0.apply(x, kern, 12, T=40, math="3xtf32").cpu() for x in X32]
    h0.close()
    torch.cuda.synchronize()
    out, errs = {}, []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                h = P.Handle(0, stream=s)
                for r in range(3):
                    y64 = h.apply(Xs[i], kern, 12, T=40)
                    y32 = h.apply(X32[i], kern, 12, T=40, math="3xtf32")
                s.synchronize()
                out[i] = (y64.cpu(), y32.cpu())
                h.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(4):
        assert torch.equal(out[i][0], ref64[i]), i
        assert torch.equal(out[i][1], ref32[i]), i
