"""The device generator (inputs/device.py) on the GPU draws the host
generator's graph bit for bit -- so the full-size configs[4] graph the bench
and the full-size tests draw on the GPU is the graph the host recipe defines."""
import numpy as np
import pytest

from inputs import graphs as G

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("n,seed", [(30000, 7), (400000, 0)])
def test_chung_lu_device_equals_host(n, seed):
    from inputs import device as D
    g = G.chung_lu(n, 2.1, 16.0, seed)
    nl, rp, c, v = D.chung_lu_csr(n, 2.1, 16.0, seed, "cuda")
    assert nl == g.n
    assert np.array_equal(rp.cpu().numpy(), g.rowptr)
    assert np.array_equal(c.cpu().numpy(), g.col)
    assert np.array_equal(v.cpu().numpy(), g.val)
