"""The C-ABI from plain C (no Python, no torch): tests/c/abi_direct.c builds
every table and runs direct / direct-cache / bitset2 / the host path through
include/fsgpu.h, checking all answers and the OutOfDomain contract.  Also:
capture of PreparedKernel.launch in a CUDA graph, and a wide table
(R >= 2^32, qbits=64) on the 64-bit bucket path."""

import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
CUDA = Path("/usr/local/cuda")


def test_c_client(cuda, tmp_path):
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler on this host")
    exe = tmp_path / "abi_direct"
    lib_dir = ROOT / "paper_1506_08620_b200"
    cmd = [gcc, "-std=c11", "-O2", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(ROOT / "tests" / "c" / "abi_direct.c"), "-L", str(lib_dir), "-l:libfsgpu.so",
           "-L", str(CUDA / "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}:{CUDA / 'lib64'}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr + res.stdout
    assert "PASS" in res.stdout


def test_launch_is_graph_capturable(cuda):
    import torch

    import paper_1506_08620_b200 as fs

    p = fs.gen_uniform_gap_partition(4097, 0.5, 1.5, seed=0, precision="single")
    z = torch.from_numpy(orc.random_queries(p.values, 1 << 20, seed=3)).to(cuda)
    out = torch.empty(z.numel(), dtype=torch.int32, device=cuda)
    for algo in ("direct", "bitset2"):
        prep = fs.prepare(algo, p)
        st = fs.new_status(cuda)
        prep.launch(z, out, st)  # warm-up outside capture (geometry cache)
        torch.cuda.synchronize()
        out.fill_(-1)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g):
                prep.launch(z, out, st)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert fs.first_bad_of(st) is None
        assert np.array_equal(out.cpu().numpy(), orc.rank_oracle(p.values, z.cpu().numpy()))
        # the status workspace stays valid across replays and reports errors
        z2 = z.clone()
        z2[12345] = float("nan")
        zz = z.clone()
        z.copy_(z2)
        g.replay()
        torch.cuda.synchronize()
        assert fs.first_bad_of(st) == 12345
        z.copy_(zz)
        g.replay()
        torch.cuda.synchronize()
        assert fs.first_bad_of(st) is None


@pytest.mark.slow
def test_wide_table_above_2_pow_32(cuda):
    """qbits=64, R >= 2^32 (K of ~17 GB): the 64-bit bucket path of build and
    search, checked against the oracle and the reference's K definition."""
    import torch

    import paper_1506_08620_b200 as fs

    xs = np.array([0.0, 2.3e-10, 0.5, 1.0], dtype=np.float64)
    p = fs.validate_partition(xs)
    h, r, _, _ = orc.compute_h_r(xs, qbits=64)
    assert r >= 1 << 32
    hg, rg, st = fs.compute_h_r(p, qbits=64)
    assert hg == h and rg == r
    with pytest.raises(fs.Overflow):
        fs.compute_h_r(p, qbits=32)
    idx = fs.build_index(p, hg, rg, qbits=64)
    f = orc.knot_buckets(xs, h)
    kd = idx.k_dev.view(torch.int32)
    for j in (0, 1, int(f[1]), int(f[1]) + 1, int(f[2]) - 1, int(f[2]), int(f[2]) + 1, r - 1, r):
        want = int(np.searchsorted(f, j, side="left"))
        assert int(kd[j].item()) & 0xFFFFFFFF == want, j
    prep = fs.prepare("direct", p, qbits=64)
    z = np.concatenate([orc.random_queries(xs, 200_000, seed=4), xs[:-1], np.nextafter(xs[1:], -np.inf)])
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))
    del idx, prep, kd
    torch.cuda.empty_cache()
