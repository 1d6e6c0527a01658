"""Multi-rank paths on ONE GPU.

Only one B200 is reachable per call, so the N>1 code paths (row shards,
the k-panel broadcast of B, max-over-ranks timing, the bench's JSON line)
are exercised with two ranks that share cuda:0 and talk over gloo.  No
kernel waits on another rank's kernel (gloo moves B through the host), so
this is safe on one GPU; NCCL over NVLink is the production transport.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["REPO"])
import numpy as np, torch, torch.distributed as dist
from paper_1710_01839_b200 import inputs, shard, PrecisionSpec
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
tok = os.environ["TOK"]
m, l, n = 200, 150, 120
a, b = inputs.gemm_inputs(tok, m, l, n, seed=9)
lo, hi = shard.row_shards(m, w, align=16)[r]
A = torch.from_numpy(np.ascontiguousarray(a[lo:hi])).cuda()
B = torch.from_numpy(b).cuda() if r == 0 else torch.zeros(b.shape, dtype=torch.float64, device="cuda")
outs = []
for panel in (None, 37):
    C = shard.broadcast_matmul(A, B, n_min=32, panel_rows=panel)
    outs.append(C.cpu().numpy())
host = shard.sharded_matmul_host(a[lo:hi], b if r == 0 else None, l, n,
                                 PrecisionSpec.parse(tok), n_min=64)
np.save(os.environ["OUT"] + f".{r}.npy", np.stack(outs + [host]))
dist.destroy_process_group()
'''


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_two_ranks_bitwise_equal_single_gpu_product(gpu, tmp_path, tok):
    import oracle
    from paper_1710_01839_b200 import inputs
    script = tmp_path / "w.py"
    script.write_text(WORKER)
    env = dict(os.environ, REPO=ROOT, TOK=tok, OUT=str(tmp_path / "c"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    parts = [np.load(str(tmp_path / f"c.{k}.npy")) for k in range(2)]
    a, b = inputs.gemm_inputs(tok, 200, 150, 120, seed=9)
    want = oracle.matmul_simple(a, b)
    for v in range(3):
        got = np.concatenate([p[v] for p in parts], axis=0)
        assert np.array_equal(got, want), v


def test_bench_two_ranks_json(gpu):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--nmin", "32", "--size", "256", "--panel", "64", "--dist-backend", "gloo",
           "--same-device", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    # strong scaling: 3 steps x 4 k-panels x (domain scan, DFMA GEMM, gated Dekker GEMM)
    assert d["gpu_launches"] == 3 * 4 * 3 and d["scaling"] == "strong"
    assert d["config"]["m"] == 256 and d["roofline"]["frac"] > 0
    # the peer-memory alternative to the broadcast (CUDA IPC between the
    # two ranks' processes, same GPU here)
    assert d["peer_mode"].get("value", 0) > 0, d["peer_mode"]
    # the reference arm under torchrun: rank 0 prints, the other exits 0
    cmd2 = cmd[:cmd.index("--gpus")] + ["--impl", "reference", "--gpus", "2", "--steps", "1",
                                        "--warmup", "0", "--size", "128", "--cpu-budget", "5"]
    r2 = subprocess.run(cmd2, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r2.returncode == 0, r2.stderr[-3000:]
    lines = [ln for ln in r2.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"


STRASSEN_WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["REPO"])
import numpy as np, torch, torch.distributed as dist
from paper_1710_01839_b200 import inputs, shard, PrecisionSpec
dist.init_process_group("gloo")
r = dist.get_rank()
torch.cuda.set_device(0)
tok, n = os.environ["TOK"], int(os.environ["N"])
a, b = inputs.gemm_inputs(tok, n, n, n, seed=12)
product, add = shard.cuda_strassen_ops(PrecisionSpec.parse(tok), 64, 32)
c = shard.strassen_distributed(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                               product=product, add=add)
np.save(os.environ["OUT"] + f".{r}.npy", c.cpu().numpy())
dist.destroy_process_group()
'''


@pytest.mark.parametrize("tok,n", [("dd", 300), ("qd", 129)])
def test_two_ranks_strassen_products_equal_single_gpu_strassen(gpu, tmp_path, tok, n):
    """The seven top-level products split over two ranks (sharing cuda:0,
    gloo moving the products through the host): C on every rank is bitwise
    the single-GPU matmul_strassen at the same cutoff."""
    import torch
    import paper_1710_01839_b200 as mp
    from paper_1710_01839_b200 import inputs
    from paper_1710_01839_b200.matrix import DenseMatrix
    out = str(tmp_path / "s")
    script = tmp_path / "ws.py"
    script.write_text(STRASSEN_WORKER)
    env = dict(os.environ, REPO=ROOT, TOK=tok, N=str(n), OUT=out)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1",
                        f"--master-port={_port()}", str(script)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    a, b = inputs.gemm_inputs(tok, n, n, n, seed=12)
    prec = mp.PrecisionSpec.parse(tok)
    want = mp.matmul_strassen(DenseMatrix(n, n, prec, a).to_device(),
                              DenseMatrix(n, n, prec, b).to_device(), 64, 32).host_array()
    for rank in range(2):
        assert np.array_equal(np.load(f"{out}.{rank}.npy"), want)


PEER_WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["REPO"])
import numpy as np, torch, torch.distributed as dist
from paper_1710_01839_b200 import inputs, shard
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
tok = os.environ["TOK"]
m, l, n = 200, 150, 120
a, b = inputs.gemm_inputs(tok, m, l, n, seed=9)
lo, hi = shard.row_shards(m, w, align=64)[r]
A = torch.from_numpy(np.ascontiguousarray(a[lo:hi])).cuda()
B = torch.from_numpy(b).cuda() if r == 0 else None
pb = shard.PeerOperand(B, src=0)
assert (r == 0) == (B is not None) and pb.shape == b.shape
C = shard.peer_matmul(A, pb, n_min=32)
torch.cuda.synchronize()
np.save(os.environ["OUT"] + f".{r}.npy", C.cpu().numpy())
pb.close()
dist.destroy_process_group()
'''


@pytest.mark.parametrize("tok", ["dd", "qd"])
def test_two_ranks_peer_memory_operand(gpu, tmp_path, tok):
    """B shared by CUDA IPC instead of broadcast: rank 1 maps rank 0's B
    (another process's allocation on the same GPU here; a peer GPU over
    NVLink on a multi-GPU box) and its GEMM reads B's tiles through the
    mapping. The stitched C is bitwise the one-process product."""
    import oracle
    from paper_1710_01839_b200 import inputs
    script = tmp_path / "p.py"
    script.write_text(PEER_WORKER)
    env = dict(os.environ, REPO=ROOT, TOK=tok, OUT=str(tmp_path / "c"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    c = np.concatenate([np.load(str(tmp_path / f"c.{k}.npy")) for k in range(2)], axis=0)
    a, b = inputs.gemm_inputs(tok, 200, 150, 120, seed=9)
    assert np.array_equal(c, oracle.matmul_simple(a, b))
