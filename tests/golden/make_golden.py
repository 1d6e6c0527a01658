#!/usr/bin/env python3
"""Generate the golden vectors in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (needs /root/reference; the GPU box does not
have it):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory, builds the
reference's Cython kernels there (``setup.py build_ext --inplace``; the
reference is read-only), imports that ``mpmm`` and records inputs and
outputs of the reference's public API:

* ``matmul_simple`` / ``matmul_block`` / ``matmul_strassen``
  (multiply.py:163-338) on seeded inputs from
  ``paper_1710_01839_b200.inputs`` (SURVEY.md s8d generators) and on the
  reference's own ``generate_test_pair`` (matrix.py:168-200);
* the ewise kernels through ``multiply._ewise`` (multiply.py:189-203);
* ``ddqd._compress4`` on QD limb vectors (pins the vectorised QD generator);
* the reference's integer known answer (tests/test_multiply.py:32-38).

Every array is stored in the reference layout (rows, cols, comps) float64.
"""

import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_PKG = "/root/reference/pkg"


def load_reference():
    scratch = os.path.join(tempfile.gettempdir(), "mpmm_ref_golden")
    if not os.path.exists(os.path.join(scratch, "src", "mpmm", "__init__.py")):
        shutil.rmtree(scratch, ignore_errors=True)
        shutil.copytree(REF_PKG, scratch)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"],
                       cwd=scratch, check=True, stdout=subprocess.DEVNULL,
                       stderr=subprocess.DEVNULL)
        # setup.py build_ext --inplace drops the module at the src root
        for f in os.listdir(scratch):
            if f.startswith("_kernels") and f.endswith(".so"):
                shutil.move(os.path.join(scratch, f), os.path.join(scratch, "src", "mpmm", f))
        for root, _, files in os.walk(os.path.join(scratch, "build")):
            for f in files:
                if f.startswith("_kernels") and f.endswith(".so"):
                    shutil.copy(os.path.join(root, f), os.path.join(scratch, "src", "mpmm", f))
    sys.path.insert(0, os.path.join(scratch, "src"))
    import mpmm
    assert mpmm.HAVE_EXT, "reference extension failed to build"
    return mpmm


def main():
    mpmm = load_reference()
    from mpmm import ddqd
    from mpmm.matrix import DenseMatrix, frobenius_norm, frobenius_rel_diff, generate_test_pair
    from mpmm.multiply import _ewise, matmul_block, matmul_simple, matmul_strassen
    from mpmm.scalar import PrecisionSpec

    sys.path.insert(0, REPO)
    from paper_1710_01839_b200 import inputs

    DD, QD = PrecisionSpec.dd(), PrecisionSpec.qd()
    prec_of = {"dd": DD, "qd": QD}

    def M(arr, prec):
        return DenseMatrix(arr.shape[0], arr.shape[1], prec, np.ascontiguousarray(arr))

    def save(name, **arrays):
        np.savez(os.path.join(HERE, name + ".npz"), **arrays)
        print("wrote", name, {k: v.shape for k, v in arrays.items()})

    # configs[0]: DD simple 128^3, seed 0 (BASELINE.json configs[0])
    a, b = inputs.gemm_inputs("dd", 128, 128, 128, seed=0)
    c = matmul_simple(M(a, DD), M(b, DD)).data
    save("cfg0_dd_simple_128", a=a, b=b, c_simple=c)

    # ragged DD blocked (reference: blocked == simple bitwise for every n_min)
    a, b = inputs.gemm_inputs("dd", 37, 45, 29, seed=11)
    cs = matmul_simple(M(a, DD), M(b, DD)).data
    cb = {f"c_block_{nm}": matmul_block(M(a, DD), M(b, DD), nm).data for nm in (1, 3, 8, 16, 64)}
    for v in cb.values():
        assert np.array_equal(v, cs)
    save("dd_ragged_37x45x29", a=a, b=b, c_simple=cs, **cb)

    # wide-exponent DD (configs[1] second input set)
    a, b = inputs.gemm_inputs("dd", 32, 48, 40, seed=12, wide=True)
    save("dd_wide_32x48x40", a=a, b=b, c_simple=matmul_simple(M(a, DD), M(b, DD)).data)

    # QD simple + blocked (configs[2] distribution)
    a, b = inputs.gemm_inputs("qd", 12, 10, 9, seed=13)
    cs = matmul_simple(M(a, QD), M(b, QD)).data
    cb = matmul_block(M(a, QD), M(b, QD), 4).data
    assert np.array_equal(cs, cb)
    save("qd_12x10x9", a=a, b=b, c_simple=cs, c_block_4=cb)

    # elementwise add/sub (multiply.py:189-203)
    for tok in ("dd", "qd"):
        x = inputs.gemm_inputs(tok, 7, 9, 1, seed=14)[0]
        y = inputs.gemm_inputs(tok, 7, 9, 1, seed=15)[0]
        p = prec_of[tok]
        save(f"{tok}_ewise_7x9", x=x, y=y,
             add=_ewise(M(x, p), M(y, p), False).data,
             sub=_ewise(M(x, p), M(y, p), True).data)

    # Strassen (multiply.py:267-338): odd padding + random inputs
    for tok, n, cut, leaf in (("dd", 33, 8, 4), ("qd", 11, 4, 4)):
        p = prec_of[tok]
        ga, gb = generate_test_pair(n, p)
        cs, cp = matmul_strassen(ga, gb, cut, leaf), matmul_simple(ga, gb)
        # matrix.py:229-294 norms, evaluated by the reference
        norms = np.array([frobenius_norm(ga), frobenius_rel_diff(cs, cp),
                          frobenius_rel_diff(ga, gb)])
        save(f"{tok}_strassen_pair{n}_c{cut}_l{leaf}", a=ga.data, b=gb.data,
             c_strassen=cs.data, c_simple=cp.data, norms=norms)
    a, b = inputs.gemm_inputs("dd", 64, 64, 64, seed=16)
    save("dd_strassen_rand64_c16_l8", a=a, b=b,
         c_strassen=matmul_strassen(M(a, DD), M(b, DD), 16, 8).data)

    # the paper's test pair (matrix.py:168-200) pins our port of the generator
    for tok, n in (("dd", 8), ("qd", 5), ("dd", 19)):
        ga, gb = generate_test_pair(n, prec_of[tok])
        save(f"{tok}_test_pair_{n}", a=ga.data, b=gb.data)

    # QD generator pin: reference ddqd._compress4 on raw limb vectors
    rng = np.random.default_rng(17)
    x0 = rng.uniform(-1, 1, 64)
    limbs = [x0] + [x0 * 2.0 ** (-53 * i) * rng.uniform(-1, 1, 64) for i in (1, 2, 3)]
    raw = np.stack(limbs, axis=-1)
    raw[5, 2] = 0.0           # exercise the zero filter
    raw[9, 1:] = 0.0
    ref = np.array([ddqd._compress4(tuple(r)) for r in raw.tolist()])
    save("qd_compress4_limbs", raw=raw, out=ref)

    # integer known answer (tests/test_multiply.py:32-38)
    ia = DenseMatrix.from_ints([[1, 2], [3, 4]], DD)
    ib = DenseMatrix.from_ints([[5, 6], [7, 8]], DD)
    save("dd_int_2x2", a=ia.data, b=ib.data, c=matmul_simple(ia, ib).data)


def edge_cases():
    """EFT-domain edge cases (eft.py:19-24, _kernels.pyx:19-29): operands
    where the reference's split TwoProd overflows (|x| >= ~2^996: NaN) or
    its error leaves the representable range (products near 2^-969,
    subnormals), signed zeros in every limb, inf and NaN.  Recorded: the
    raw kernel output of the reference's ext backend (simple rows and block
    cells, which never raise) and whether the public matmul_simple raises
    RangeError (multiply.py:124-127)."""
    mpmm = load_reference()
    from mpmm import backend
    from mpmm.errors import RangeError
    from mpmm.matrix import DenseMatrix
    from mpmm.multiply import matmul_simple, matmul_strassen
    from mpmm.scalar import PrecisionSpec

    sys.path.insert(0, REPO)
    from paper_1710_01839_b200 import inputs

    kern = backend.kernels()
    assert kern.NAME == "ext"
    DD, QD = PrecisionSpec.dd(), PrecisionSpec.qd()

    def M(arr, prec):
        return DenseMatrix(arr.shape[0], arr.shape[1], prec, np.ascontiguousarray(arr))

    def record(name, a, b, prec, n_min=4):
        comps = a.shape[2]
        pre = "dd" if comps == 2 else "qd"
        m, n = a.shape[0], b.shape[1]
        cs = np.zeros((m, n, comps))
        getattr(kern, f"{pre}_simple_rows")(a, b, cs, 0, m)
        cb = np.zeros((m, n, comps))
        cells = (-(-m // n_min)) * (-(-n // n_min))
        getattr(kern, f"{pre}_block_cells")(a, b, cb, n_min, 0, cells)
        assert np.array_equal(cs, cb, equal_nan=True)
        try:
            matmul_simple(M(a, prec), M(b, prec))
            raises = 0
        except RangeError:
            raises = 1
        np.savez(os.path.join(HERE, name + ".npz"), a=a, b=b, c=cs,
                 raises=np.array(raises), n_min=np.array(n_min))
        print("wrote", name, "raises" if raises else "ok",
              "nan" if np.isnan(cs).any() else "")

    m, l, n = 6, 7, 5
    base_a, base_b = inputs.gemm_inputs("dd", m, l, n, seed=40)

    def dd_scaled(ea, eb, rows=(0, 2), cols=(1, 3)):
        a, b = base_a.copy(), base_b.copy()
        for i in rows:
            a[i] = np.ldexp(a[i], ea)
        for j in cols:
            b[:, j] = np.ldexp(b[:, j], eb)
        return a, b

    # split overflow side: 2^995 (inside the reference's range), 2^996 and
    # 2^996.9 (the boundary), 2^1000 (overflowed split -> NaN)
    for tag, ea, eb in (("big995", 995, -990), ("big996", 996, -996), ("big997", 997, -997),
                        ("big1000", 1000, -1000)):
        a, b = dd_scaled(ea, eb)
        record(f"edge_dd_{tag}", a, b, DD)
    a, b = dd_scaled(996, -996)
    a[0, 0] = [1.99 * 2.0 ** 996, 2.0 ** 943]
    record("edge_dd_big996_9", a, b, DD)
    # error underflow side: products near 2^-969, subnormal operands
    for tag, ea, eb in (("tiny969", -500, -470), ("tiny1000", -520, -480),
                        ("tiny1040", -540, -500)):
        a, b = dd_scaled(ea, eb)
        record(f"edge_dd_{tag}", a, b, DD)
    a, b = base_a.copy(), base_b.copy()
    a[1, :, 0] = np.ldexp(np.abs(a[1, :, 0]) + 0.5, -1060)   # subnormal high words
    a[1, :, 1] = 0.0
    b[:, 2] = np.ldexp(b[:, 2], -3)
    record("edge_dd_subnormal", a, b, DD)
    # signed zeros, inf, NaN
    a, b = base_a.copy(), base_b.copy()
    a[0] = 0.0
    a[1] = -0.0
    a[2, :, 1] = -0.0
    b[:, 0] = -0.0
    b[3, :, 1] = 0.0
    b[4] = [-0.0, 0.0]
    record("edge_dd_zeros", a, b, DD)
    a, b = base_a.copy(), base_b.copy()
    a[2, 3] = [np.inf, 0.0]
    b[1, 4] = [np.nan, 0.0]
    record("edge_dd_inf_nan", a, b, DD)
    # a product that overflows, finite operands (2^600 * 2^500)
    a, b = dd_scaled(600, 500)
    record("edge_dd_overflow", a, b, DD)

    # QD: signed-zero limbs in every position, big and tiny limbs
    qa, qb = inputs.gemm_inputs("qd", 5, 6, 4, seed=41)
    a, b = qa.copy(), qb.copy()
    a[0, :, 3] = 0.0
    a[1, :, 2:] = -0.0
    a[2, 0] = [0.0, -0.0, 0.0, -0.0]
    b[:, 1, 1:] = 0.0
    b[2] = -0.0
    b[3, :, 3] = -0.0
    record("edge_qd_zeros", a, b, QD, n_min=2)
    a, b = qa.copy(), qb.copy()
    a[0] = np.ldexp(a[0], 997)
    b[:, 0] = np.ldexp(b[:, 0], -997)
    record("edge_qd_big997", a, b, QD, n_min=2)
    a, b = qa.copy(), qb.copy()
    a[1] = np.ldexp(a[1], -300)
    b[:, 2] = np.ldexp(b[:, 2], -500)
    record("edge_qd_tiny", a, b, QD, n_min=2)

    # Strassen on large operands: the leaf operands are quadrant sums
    sa, sb = inputs.gemm_inputs("dd", 16, 16, 16, seed=42)
    sa = np.ldexp(sa, 993)
    sb = np.ldexp(sb, -993)
    cs = matmul_strassen(M(sa, DD), M(sb, DD), 4, 2)
    np.savez(os.path.join(HERE, "edge_dd_strassen_big.npz"), a=sa, b=sb, c=cs.data)
    print("wrote edge_dd_strassen_big")


def scalar_cases():
    """The reference's host scalar algebra (scalar.py:95-251 over ddqd.py):
    add/sub/mul/div/sqrt on seeded DD and QD pairs, and the literal
    constructors, recorded for tests/test_host_logic.py."""
    load_reference()
    from mpmm.scalar import PrecisionSpec, Scalar, scalar_sqrt

    sys.path.insert(0, REPO)
    from paper_1710_01839_b200 import inputs

    out = {}
    for tok in ("dd", "qd"):
        prec = PrecisionSpec.parse(tok)
        a, b = inputs.gemm_inputs(tok, 1, 40, 1, seed=70)
        xs = [Scalar(prec, tuple(float(c) for c in a[0, k])) for k in range(40)]
        ys = [Scalar(prec, tuple(float(c) for c in b[k, 0])) for k in range(40)]
        out[f"{tok}_x"] = np.array([x.payload for x in xs])
        out[f"{tok}_y"] = np.array([y.payload for y in ys])
        for name, fn in (("add", lambda x, y: x + y), ("sub", lambda x, y: x - y),
                         ("mul", lambda x, y: x * y), ("div", lambda x, y: x / y)):
            out[f"{tok}_{name}"] = np.array([fn(x, y).payload for x, y in zip(xs, ys)])
        out[f"{tok}_sqrt"] = np.array([scalar_sqrt(x if x.payload[0] >= 0 else -x).payload
                                       for x in xs])
        out[f"{tok}_lits"] = np.array([Scalar.from_str("0.1", prec).payload,
                                       Scalar.from_str("-3.14159265358979323846264338327950288",
                                                       prec).payload,
                                       Scalar.from_int(2 ** 60 + 1, prec).payload,
                                       Scalar.from_int(-(3 ** 70), prec).payload])
    np.savez(os.path.join(HERE, "scalar_ops.npz"), **out)
    print("wrote scalar_ops", sorted(out))


if __name__ == "__main__":
    if "--edge" in sys.argv:
        edge_cases()
    elif "--scalar" in sys.argv:
        scalar_cases()
    else:
        main()
        edge_cases()
        scalar_cases()
