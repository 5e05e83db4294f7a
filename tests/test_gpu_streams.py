"""The C-ABI's threading contract: stream-ordered, safe from
several host threads on distinct streams.  Each thread runs the tensor-core
product and an elementwise operator on its own stream, concurrently, and
must get exactly the bits of a serial run."""
import threading

import numpy as np
import pytest

from mcgen import assert_bits, split

pytestmark = pytest.mark.gpu


def test_concurrent_streams_match_serial_results():
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(90)
    jobs = []
    for t in range(4):
        m, k, n = 300 + 37 * t, 700, 200 + 11 * t
        x = torch.from_numpy(split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)).cuda()
        w = torch.from_numpy(rng.uniform(-1, 1, (k, n)).astype(np.float32)).cuda()
        y = torch.from_numpy(split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)).cuda()
        jobs.append((x, w, y))
    serial = [(mcf.mm_mcn(x, w, plan=mcf.FAST).cpu().numpy(), mcf.add_mcn(x, y).cpu().numpy()) for x, w, y in jobs]
    results = [None] * len(jobs)
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                x, w, y = jobs[i]
                outs = []
                for _ in range(3):
                    outs.append((mcf.mm_mcn(x, w, plan=mcf.FAST), mcf.add_mcn(x, y)))
                s.synchronize()
                results[i] = [(a.cpu().numpy(), b.cpu().numpy()) for a, b in outs]
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i, (mm_s, add_s) in enumerate(serial):
        for mm_c, add_c in results[i]:
            assert_bits(mm_c, mm_s, f"thread {i} mm")
            assert_bits(add_c, add_s, f"thread {i} add")


def test_errors_are_per_thread_and_reference_worded():
    """mcf_last_error is thread-local and carries the reference's messages."""
    import torch

    import paper_2207_08867_b200 as mcf

    x = torch.zeros((3, 5, 2), dtype=torch.float32, device="cuda")
    w = torch.zeros((2, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError, match=r"\(3,5\)"):
        mcf.mm_mcn(x, w)
    with pytest.raises(mcf.UnsupportedOperation):
        mcf.mm_mcn(x, torch.zeros((5, 4, 2), dtype=torch.float32, device="cuda"))
    bad = torch.zeros((4, 9), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError, match="1 <= nc <= 8"):
        mcf.square_mcn(bad)


def test_reserved_product_runs_under_stream_capture():
    """mcf_fast_mm_reserve grows the stream's workspace ahead of time, so the
    FAST product allocates nothing and can be captured into a CUDA graph on a
    stream that has never run it; the replay gives the bits of a direct call."""
    import torch

    import paper_2207_08867_b200 as mcf

    lib = mcf.lib()
    rng = np.random.default_rng(91)
    m, k, n = 512, 1024, 384
    x = torch.from_numpy(split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)).cuda()
    w = torch.from_numpy(rng.uniform(-1, 1, (k, n)).astype(np.float32)).cuda()
    want = mcf.mm_mcn(x, w, plan=mcf.FAST).cpu().numpy()
    out = torch.zeros((m, n, 2), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    assert lib.mcf_fast_mm_reserve(m, k, n, 1, s.cuda_stream) == 0, lib.mcf_last_error()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            rc = lib.mcf_bmm_mcn(mcf.B32, x.data_ptr(), 2, w.data_ptr(), 1, m, k, n, 0, out.data_ptr(), mcf.FAST, 1,
                                 torch.cuda.current_stream().cuda_stream)
            assert rc == 0, lib.mcf_last_error()
        g.replay()
        s.synchronize()
    assert_bits(out.cpu().numpy(), want, "captured FAST product")
    assert lib.mcf_fast_mm_reserve(8, 1 << 20, 8, 1, 0) == 2  # MCF_ERR_UNSUPPORTED: outside the scheme
