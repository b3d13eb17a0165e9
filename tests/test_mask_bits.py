"""The bit-packed mask layout of disc_frame::mask_bits (include/disc.h): pixel p = v*W + u of plane s
is bit p % 32 of little-endian word p / 32, bits past H*W zero.  synth.pack_mask_bits (the input
generator's packer, used by the tests and bench.py) against numpy's packbits on random planes,
ragged H*W included."""
import numpy as np
import pytest
import torch

from synth import pack_mask_bits


@pytest.mark.parametrize("S,H,W", [(1, 1, 1), (3, 7, 13), (5, 48, 64), (2, 239, 317), (4, 32, 1)])
def test_pack_matches_numpy_packbits(S, H, W):
    rng = np.random.default_rng(S * 1000 + H * 10 + W)
    m = (rng.random((S, H, W)) < 0.4).astype(np.uint8) * rng.integers(1, 256, (S, H, W)).astype(np.uint8)
    words = pack_mask_bits(torch.from_numpy(m)).numpy().view(np.uint32)
    ref = np.packbits(m.reshape(S, -1) != 0, axis=1, bitorder="little")
    ref = np.pad(ref, ((0, 0), (0, (-ref.shape[1]) % 4))).view("<u4")
    assert words.shape == (S, (H * W + 31) // 32)
    assert np.array_equal(words, ref)


def test_every_pixel_is_its_own_bit():
    """One pixel set at a time: exactly bit p % 32 of word p / 32."""
    H, W = 5, 11
    for p in range(H * W):
        m = torch.zeros(1, H, W, dtype=torch.uint8)
        m.view(-1)[p] = 1
        w = pack_mask_bits(m).numpy().view(np.uint32)[0]
        expect = np.zeros_like(w)
        expect[p // 32] = np.uint32(1) << np.uint32(p % 32)
        assert np.array_equal(w, expect), p
