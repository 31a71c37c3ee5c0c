"""fs_all_finite (the device finiteness check behind ScoreMatrix / DampedSystem validation)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "float64", "complex64", "complex128"])
@pytest.mark.parametrize("shape", [(1,), (7,), (3, 5), (33, 1001), (1024, 4099)])
def test_all_finite_finds_every_bad_entry(dtype, shape):
    from paper_2310_17556_b200 import _lib
    dev = torch.device("cuda", 0)
    t = torch.zeros(shape, dtype=getattr(torch, dtype), device=dev)
    assert _lib.all_finite(t)
    rng = np.random.Generator(np.random.PCG64(sum(shape)))
    for bad in (float("nan"), float("inf"), -float("inf")):
        for _ in range(3):
            idx = tuple(int(rng.integers(0, s)) for s in shape)
            u = t.clone()
            u[idx] = bad if not u.is_complex() else complex(0.0, bad)
            assert not _lib.all_finite(u), (idx, bad)


@pytest.mark.gpu
def test_all_finite_respects_the_leading_dimension():
    """Pad columns beyond the logical width are never read (ScoreMatrix pads rows to 16 bytes)."""
    from paper_2310_17556_b200 import _lib
    dev = torch.device("cuda", 0)
    buf = torch.full((17, 40), float("nan"), dtype=torch.float32, device=dev)
    buf[:, :37] = 1.0
    assert _lib.all_finite(buf[:, :37])
    buf[16, 36] = float("inf")
    assert not _lib.all_finite(buf[:, :37])
