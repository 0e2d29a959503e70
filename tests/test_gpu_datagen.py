"""The device copy of the input generators matches the host one bit for bit
(the multi-GPU configuration generates its inputs on the GPU; the oracle side
regenerates samples on the host)."""
import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_bytes_match_host():
    t = torch.empty(4096 * 8, dtype=torch.uint8, device="cuda")
    datagen.random_bytes_cuda(t, 0x501, offset=8 * 1000)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), datagen.random_bytes(4096 * 8, 0x501, offset=8 * 1000))


def test_feistel_matches_host_and_permutes():
    n = 5000
    d = datagen.feistel_cuda(n, 0, n, 0x502).cpu().numpy().astype(np.uint64)
    assert np.array_equal(d, datagen.feistel(n, 0, n, 0x502))
    assert np.array_equal(np.sort(d), np.arange(n, dtype=np.uint64))
    big = datagen.feistel_cuda(1 << 30, 12345, 1000, 0x502).cpu().numpy().astype(np.uint64)
    assert np.array_equal(big, datagen.feistel(1 << 30, 12345, 1000, 0x502))
