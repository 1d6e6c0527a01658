"""tcgen05 residue GEMMs (csrc/tc_i8.cu) against cuBLASLt's exact int8
GEMM reduced on the host: R_t = (A_t Bt_t^T) mod p_t, bit for bit."""
import numpy as np
import pytest

from paper_1710_01839_b200 import _cuda, tensor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k,batch", [(128, 256, 128, 1), (256, 512, 384, 3),
                                         (1024, 1024, 1024, 5), (128, 256, 4096, 54)])
def test_residue_gemm_matches_cublaslt(gpu, m, n, k, batch):
    import torch
    g = torch.Generator().manual_seed(m + n + k + batch)
    A = torch.randint(-128, 128, (batch, m, k), generator=g, dtype=torch.int8).cuda()
    B = torch.randint(-128, 128, (batch, n, k), generator=g, dtype=torch.int8).cuda()
    R = torch.empty((batch, m, n), dtype=torch.uint8, device="cuda")
    G = torch.empty((batch, m, n), dtype=torch.int32, device="cuda")
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _cuda.residue_gemm_dev(m, n, k, batch, A.data_ptr(), B.data_ptr(), R.data_ptr(), s)
    _cuda.int8_gemm_batched_dev(m, n, k, batch, A.data_ptr(), B.data_ptr(), G.data_ptr(),
                                ws.data_ptr(), 64 << 20, s)
    torch.cuda.synchronize()
    p = np.array(tensor.MODULI[:batch], dtype=np.int64).reshape(-1, 1, 1)
    want = np.mod(G.cpu().numpy().astype(np.int64), p).astype(np.uint8)
    assert np.array_equal(R.cpu().numpy(), want)


def test_residue_gemm_rejects_bad_shapes(gpu):
    with pytest.raises(ValueError):
        _cuda.residue_gemm_dev(100, 256, 128, 1, 0, 0, 0)


@pytest.mark.parametrize("variant", ["tile", "pair"])
def test_residue_gemm_kernel_variants(gpu, variant):
    """The one-tile-per-CTA kernel and the cluster-pair (B multicast) kernel,
    forced through MPMM_TC_KERNEL in a child process, against cuBLASLt."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MPMM_TC_KERNEL=variant)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_tcgen05.py"),
                        "-k", "matches_cublaslt"], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
