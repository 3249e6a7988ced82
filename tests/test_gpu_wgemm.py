"""K7, the tcgen05 weight-streaming GEMM for the M <= 256 projections
(csrc/gemm_tc.cu; chosen per decode bucket and shape against the best
cuBLASLt plan at start-up, CS_WGEMM=2 by default; CS_WGEMM=1 forces it):
its output against cuBLASLt on seeded bf16 operands over the decode
bucket sizes, every cluster size it launches (K split 1..8) and fp32 output,
and a whole forward (prefill, decode CUDA graphs) with K7 against the fp32
oracle. Tolerance: bf16 output rounding (|K7 - cuBLAS| <= 1e-2 x max |Y|)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from helpers import DECISIVE_AGREE, Driver, decisive_rows, logit_bound

pytestmark = pytest.mark.gpu


def _bench(eng, M, N, K):
    a, b, d, r = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    cs.engine._check(cs.lib().cs_bench_gemm(eng._h, M, N, K, 2, C.byref(a), C.byref(b), C.byref(d), C.byref(r)))
    return d.value, r.value


@pytest.fixture(scope="module", params=["stream-k", "cluster"])
def eng(request):
    """K7 in its default cluster split-K mode (CS_K7_SK=0: the K splits of a
    feature tile reduced through DSMEM) and in the stream-K mode (CS_K7_SK=1:
    one persistent CTA per SM over equal (tile, K-chunk) ranges, cut tiles
    folded from fp32 partials)."""
    old = os.environ.get("CS_K7_SK")
    os.environ["CS_K7_SK"] = "1" if request.param == "stream-k" else "0"
    try:
        e = cs.Engine(cs.model_config("tiny", gpu_kv_capacity=1 << 26))
    finally:
        if old is None:
            os.environ.pop("CS_K7_SK")
        else:
            os.environ["CS_K7_SK"] = old
    yield e
    e.close()


@pytest.mark.parametrize("M", [1, 8, 17, 64, 128, 200, 256])
@pytest.mark.parametrize("N,K", [(6144, 4096), (4096, 14336), (128, 64), (28672, 4096), (512, 256), (128256, 4096)])
def test_k7_matches_cublas(eng, M, N, K):
    diff, ref = _bench(eng, M, N, K)
    assert ref > 0
    assert diff <= 1e-2 * ref, (diff, ref)


def test_forward_with_k7_matches_oracle(monkeypatch):
    monkeypatch.setenv("CS_WGEMM", "1")
    drv = Driver(cs.model_config("tiny", num_layers=2, hidden=512, n_heads=8, n_kv_heads=4, head_dim=64, ffn=1024,
                                 vocab=1024, max_batched_tokens=1024))
    agree, rows = 0, 0
    try:
        for r in range(8):
            drv.add(r, 12 + 9 * r, online=r < 2)
        plans = [[(r, None) for r in range(8)]] * 5
        for plan in plans:
            info, lg, ref = drv.step(plan)
            bound = logit_bound(ref)
            assert float(np.max(np.abs(lg - ref))) <= bound
            ok, dec = decisive_rows(lg, ref, bound)
            agree += ok
            rows += dec
    finally:
        drv.close()
    assert agree >= DECISIVE_AGREE * rows, (agree, rows)  # decisive rows over the run
    assert os.environ.get("CS_WGEMM") == "1"
