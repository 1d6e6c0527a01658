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


if __name__ == "__main__":
    main()
