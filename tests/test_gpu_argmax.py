"""The sampled ids (argmax_kernel: 16 CTAs per row folding (ordered value,
~id) keys with atomicMax; keys re-armed by the final RMSNorm) against numpy's
argmax of the same device logits, exactly (ties -> lowest id, as np.argmax),
through prefill and decode-graph steps, for a vocabulary the 16-byte-load
path takes (1024) and one it does not (1001, vocab % 4 != 0)."""
import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from helpers import Driver

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("vocab", [1024, 1001])
def test_sampled_ids_are_the_argmax_of_the_logits(vocab):
    drv = Driver(cs.model_config("tiny", num_layers=2, vocab=vocab))
    try:
        for r in range(6):
            drv.add(r, 10 + 7 * r, online=r < 2)
        for _ in range(4):  # prefill, then decode steps (CUDA graphs)
            info, lg, ref = drv.step([(r, None) for r in range(6)])
            assert info.n_outputs == 6
            assert info.tokens == [int(i) for i in np.argmax(lg, axis=1)]
    finally:
        drv.close()
