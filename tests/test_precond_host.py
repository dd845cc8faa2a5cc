"""Host-side pieces of the pluggable preconditioners, no GPU needed.

* BlockJacobiPreconditioner's dense diagonal blocks (what the device factorises)
  equal the blocks of the dense matrix, including a short padded last block;
* the reference-side block-Jacobi Preconditioner subclass (oracle/_ref, driven
  through the unmodified reference mpk_chebyshev: z_0 = M^-1 r) applies exactly
  those blocks' inverse (to rounding).
"""
import numpy as np
import pytest


def _dense(o):
    a = np.zeros((o.n, o.n))
    for i in range(o.n):
        for k in range(o.rowptr[i], o.rowptr[i + 1]):
            a[i, o.col[k]] += o.val[k]
    return a


@pytest.mark.parametrize("bs", [1, 3, 4, 7])
def test_block_extraction(port, bs):
    import paper_2603_09790_b200 as cs
    o = port.poisson27(5, 4, 3)  # n = 60: a short last block for bs = 7
    m = cs.BlockJacobiPreconditioner(cs.CsrMatrix(o.n, o.rowptr, o.col, o.val), bs)
    a = _dense(o)
    nb = (o.n + bs - 1) // bs
    assert m.blocks.shape == (nb, bs, bs)
    for b in range(nb):
        r0, r1 = b * bs, min(o.n, b * bs + bs)
        want = np.eye(bs)
        want[:r1 - r0, :r1 - r0] = a[r0:r1, r0:r1]
        # blocks[b] is the column-major bs x bs block: element (i, j) at [b, j, i]
        assert np.array_equal(m.blocks[b].T, want)


@pytest.mark.parametrize("bs", [2, 4, 6])
def test_reference_subclass_applies_block_inverse(ref, port, bs):
    o = port.poisson27(6, 5, 4)
    a = _dense(o)
    r = np.random.default_rng(bs).standard_normal(o.n)
    z, _ = ref.mpk(o, r, 1, 0.1, 1.5, precond=100 + bs)
    want = np.empty(o.n)
    for r0 in range(0, o.n, bs):
        r1 = min(o.n, r0 + bs)
        want[r0:r1] = np.linalg.solve(a[r0:r1, r0:r1], r[r0:r1])
    np.testing.assert_allclose(z[0], want, rtol=1e-13, atol=1e-15)


def test_device_preconditioner_callback_is_a_c_function():
    import ctypes as C

    import paper_2603_09790_b200 as cs

    class Scale(cs.DevicePreconditioner):
        def device_apply(self, in_ptr, out_ptr, n, stream):
            self.seen = (in_ptr, out_ptr, n, stream)

    s = Scale()
    cb = s._c_callback()
    # called through its C function pointer, the way the library calls it
    fn = C.cast(cb, C.c_void_p).value
    proto = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
    assert proto(fn)(None, 16, 32, 7, 99) == 0
    assert s.seen == (16, 32, 7, 99)
