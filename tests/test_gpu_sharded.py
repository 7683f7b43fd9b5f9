"""The row-sharded driver with the CUDA rank backend (libcfb200) through NCCL.

Only one GPU is available to the tests, so the process group has world_size 1:
the reduce-scatter / all-gather are identities, but every kernel and the whole
driver path (partition, partial A^T h, cf_column_update with global counts,
x all-gather into the plan's buffer, cf_plan_row_step, report parts) run.
The multi-rank exchange itself is covered on CPU by tests/test_sharded.py.
"""

import os
import socket

import numpy as np
import pytest

import oracle
from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,mu", [("lp", 1.0), ("socp4", 0.6)])
def test_sharded_cuda_backend_matches_oracle(nccl_group, kind, mu):
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve
    from paper_2203_05027_b200.sharded import solve_sharded

    p = generate(GenSpec(60, 160, 0.05, kind, seed=41))
    cfg = SolverConfig(mu=mu, eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=3000)
    res = solve_sharded(p, cfg)
    ox, olam, otrace, _ = oracle.solve(p, cfg)
    assert [r.iter for r in res.trace] == [r["iter"] for r in otrace]
    assert [r.status for r in res.trace] == [r["status"] for r in otrace]
    assert rel_err(res.x, ox) <= 1e-8 and rel_err(res.lam, olam) <= 1e-8
    ref = solve(p, cfg)
    assert res.report.iter == ref.report.iter
    np.testing.assert_allclose(res.report.pobj, ref.report.pobj, rtol=1e-10)


def test_sharded_large_instance_matches_single_plan(nccl_group):
    """20M nonzeros (the size where an unordered plan stream raced torch's copies):
    the sharded loop on torch's default stream equals the single-plan iteration bit for bit."""
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device_shard
    from paper_2203_05027_b200.sharded import CudaRankBackend, run_sharded

    st = torch.cuda.current_stream()
    plan, rc, cc, cs, bn, cn, cones = generate_device_shard(1_000_000, 2_000_000, 1e-5, "lp", 0, 0, 1,
                                                            stream=st.cuda_stream)
    iters = 8
    plan.set_state(1.0, None, export=False)
    plan.iterate(1.0, iters)
    ref = plan.get_state(want_yg=False)
    plan.set_state(1.0, None, export=False)
    be = CudaRankBackend.from_plan(plan, cc[0], cc[1], cs, cones)
    cfg = SolverConfig(max_iters=iters, check_every=5, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    res = run_sharded(be, rc, cc, cfg, bn, cn)
    assert np.array_equal(res.x, ref["x"])
    assert np.array_equal(res.lam, ref["lam"])
    be.close()


def test_sharded_overlapped_reduce_equals_reduce_scatter(nccl_group):
    """Slice-by-slice column pass + per-slice reduce == whole pass + reduce-scatter (bit for bit)."""
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device_shard
    from paper_2203_05027_b200.sharded import CudaRankBackend, run_sharded

    st = torch.cuda.current_stream()
    plan, rc, cc, cs, bn, cn, cones = generate_device_shard(20_000, 40_000, 5e-4, "lp", 3, 0, 1,
                                                            stream=st.cuda_stream)
    cfg = SolverConfig(max_iters=60, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    out = []
    for overlap in (False, True):
        plan.set_state(1.0, None, export=False)
        be = CudaRankBackend.from_plan(plan, cc[0], cc[1], cs, cones)
        out.append(run_sharded(be, rc, cc, cfg, bn, cn, overlap_reduce=overlap))
    assert np.array_equal(out[0].x, out[1].x) and np.array_equal(out[0].lam, out[1].lam)
    assert [r.prim_res_2 for r in out[0].trace] == [r.prim_res_2 for r in out[1].trace]
    plan.close()


def test_column_range_pass_covers_every_column_once(nccl_group):
    """cf_apply_At_cols over consecutive ranges == cf_apply_At, for cuts inside tiles too."""
    import ctypes

    import torch

    from paper_2203_05027_b200 import _lib
    from paper_2203_05027_b200.devgen import generate_device

    inst = generate_device(30_000, 90_000, 4e-4, "lp", seed=5)
    plan = inst.plan
    y = torch.randn(inst.m, dtype=torch.float64, device="cuda")
    full = torch.empty(inst.n, dtype=torch.float64, device="cuda")
    plan.apply_At(y.data_ptr(), full.data_ptr())
    parts = torch.full((inst.n,), float("nan"), dtype=torch.float64, device="cuda")
    cuts = [0, 1, 777, 30_000, 30_001, 61_234, inst.n]
    L = _lib.lib()
    for a, b in zip(cuts[:-1], cuts[1:]):
        _lib.check(L.cf_apply_At_cols(plan.handle, ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(parts.data_ptr()),
                                      a, b))
    torch.cuda.synchronize()
    assert torch.equal(parts, full)
    plan.close()


def test_sharded_with_column_bands_matches_single_plan(nccl_group, monkeypatch):
    """Banded plans (h split into row bands) through the sharded driver: the range pass
    falls back to the whole banded pass and the result equals the single-plan iteration."""
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device_shard
    from paper_2203_05027_b200.sharded import CudaRankBackend, run_sharded

    monkeypatch.setenv("CF_BAND_MB", "0.05")
    st = torch.cuda.current_stream()
    plan, rc, cc, cs, bn, cn, cones = generate_device_shard(30_000, 60_000, 3e-4, "lp", 2, 0, 1,
                                                            stream=st.cuda_stream)
    iters = 40
    plan.set_state(1.0, None, export=False)
    plan.iterate(1.0, iters)
    ref = plan.get_state(want_yg=False)
    plan.set_state(1.0, None, export=False)
    be = CudaRankBackend.from_plan(plan, cc[0], cc[1], cs, cones)
    cfg = SolverConfig(max_iters=iters, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    res = run_sharded(be, rc, cc, cfg, bn, cn)
    assert np.array_equal(res.x, ref["x"]) and np.array_equal(res.lam, ref["lam"])
    be.close()


@pytest.mark.parametrize("kind,mu", [("lp", 1.0), ("socp4", 0.6)])
def test_column_sharded_cuda_backend_matches_oracle(nccl_group, kind, mu):
    """Column sharding with the CUDA backend (cf_plan_col_step, cf_apply_A_async, the
    all-reduce of A x, cf_plan_row_update, global row norms) reaches the oracle's solve."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate
    from paper_2203_05027_b200.sharded import solve_col_sharded

    p = generate(GenSpec(120, 400, 0.04, kind, seed=17))
    cfg = SolverConfig(mu=mu, max_iters=3000, eps_prim=1e-5, eps_dual=1e-5, eps_gap=1e-5)
    res = solve_col_sharded(p, cfg)
    ox, olam, otrace, _ = oracle.solve(p, cfg)
    assert [r.iter for r in res.trace] == [r["iter"] for r in otrace]
    assert res.report.status == otrace[-1]["status"]
    assert rel_err(res.x, ox) <= 1e-8 and rel_err(res.lam, olam) <= 1e-8


@pytest.mark.parametrize("kind", ["lp", "socp4"])
def test_sharded_p2p_step_equals_nccl_step(nccl_group, kind):
    """The fused peer-memory step (cf_column_update_p2p on IPC-exported buffers; with one
    rank the peers are the rank itself) == reduce-scatter + update + all-gather, bit for bit."""
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device_shard
    from paper_2203_05027_b200.sharded import CudaRankBackend, run_sharded

    st = torch.cuda.current_stream()
    plan, rc, cc, cs, bn, cn, cones = generate_device_shard(20_000, 40_000, 5e-4, kind, 3, 0, 1,
                                                            stream=st.cuda_stream)
    cfg = SolverConfig(max_iters=60, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    out = []
    for p2p in (False, True):
        plan.set_state(1.0, None, export=False)
        be = CudaRankBackend.from_plan(plan, cc[0], cc[1], cs, cones)
        out.append(run_sharded(be, rc, cc, cfg, bn, cn, p2p=p2p))
        be.disable_p2p()
    assert np.array_equal(out[0].x, out[1].x) and np.array_equal(out[0].lam, out[1].lam)
    assert out[0].trace == out[1].trace
    plan.close()


@pytest.mark.parametrize("cones", [False, True])
def test_p2p_update_kernel_two_sources(cones):
    """cf_column_update_p2p with two partial sources and two x destinations (here both on
    this GPU) == cf_column_update on their rank-order sum, and every destination gets x+."""
    import ctypes

    import torch

    from paper_2203_05027_b200 import _lib

    L = _lib.lib()
    n = 12_000
    g = torch.Generator(device="cuda")
    g.manual_seed(7)

    def rnd():
        return torch.randn(n, generator=g, device="cuda", dtype=torch.float64)

    a, b, c, x, z, d = rnd(), rnd(), rnd(), rnd(), rnd(), rnd()
    cnt = torch.randint(0, 20, (n,), generator=g, device="cuda").double()
    cone_ptr = torch.arange(0, n + 1, 4, dtype=torch.int32, device="cuda") if cones else None
    nb = n // 4 if cones else 0

    def p(t):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    x1, z1, d1 = x.clone(), z.clone(), d.clone()
    ath = a + b
    _lib.check(L.cf_column_update(n, p(ath), p(cnt), p(c), p(x1), p(z1), p(d1), 0.7, nb, p(cone_ptr), None))
    x2, z2, d2 = x.clone(), z.clone(), d.clone()
    dst1, dst2 = torch.zeros(n, dtype=torch.float64, device="cuda"), torch.full((n,), 5.0, dtype=torch.float64,
                                                                                 device="cuda")
    parts = torch.tensor([a.data_ptr(), b.data_ptr()], dtype=torch.int64, device="cuda")
    dsts = torch.tensor([dst1.data_ptr(), dst2.data_ptr()], dtype=torch.int64, device="cuda")
    _lib.check(L.cf_column_update_p2p(n, p(parts), 2, p(cnt), p(c), p(x2), p(z2), p(d2), 0.7, nb, p(cone_ptr),
                                      p(dsts), 2, None))
    torch.cuda.synchronize()
    assert torch.equal(x1, x2) and torch.equal(z1, z2) and torch.equal(d1, d2)
    assert torch.equal(dst1, x2) and torch.equal(dst2, x2)


def test_ipc_buffer_opens_in_another_process():
    """cf_ipc_alloc's handle opens in another process (cf_ipc_open) and shows the same bytes."""
    import ctypes
    import subprocess
    import sys

    import torch

    from paper_2203_05027_b200 import _lib
    from paper_2203_05027_b200.sharded import _DevArray

    L = _lib.lib()
    ptr, h = ctypes.c_void_p(), ctypes.create_string_buffer(64)
    _lib.check(L.cf_ipc_alloc(8 * 64, ctypes.byref(ptr), h))
    try:
        view = torch.as_tensor(_DevArray(ptr.value, 64), device="cuda")
        view.copy_(torch.arange(64, dtype=torch.float64, device="cuda") * 1.5)
        torch.cuda.synchronize()
        child = (
            "import ctypes, sys, torch\n"
            "from paper_2203_05027_b200 import _lib\n"
            "from paper_2203_05027_b200.sharded import _DevArray\n"
            "torch.cuda.init()\n"
            "L = _lib.lib(); ptr = ctypes.c_void_p()\n"
            "_lib.check(L.cf_ipc_open(ctypes.create_string_buffer(bytes.fromhex(sys.argv[1]), 64), ctypes.byref(ptr)))\n"
            "v = torch.as_tensor(_DevArray(ptr.value, 64), device='cuda').cpu()\n"
            "print(float(v.sum()), float(v[63]))\n"
            "L.cf_ipc_close(ptr)\n")
        out = subprocess.run([sys.executable, "-c", child, h.raw.hex()], capture_output=True, text=True, timeout=300,
                             cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert out.returncode == 0, out.stderr[-2000:]
        total, last = (float(v) for v in out.stdout.split())
        assert total == float(sum(1.5 * k for k in range(64))) and last == 94.5
    finally:
        L.cf_ipc_free(ptr)


_MC = {}


def _mc_supported():
    """The device reports multicast support AND the driver creates a multicast object here.
    (The single-GPU boxes of this pool report CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 1
    but refuse cuMulticastCreate with CUDA_ERROR_INVALID_VALUE: no NVSwitch fabric team;
    scratch/mc_probe.cu, profiles/r02_probes.md.)"""
    import ctypes

    from paper_2203_05027_b200 import _lib

    if "ok" not in _MC:
        s = ctypes.c_int(0)
        _lib.check(_lib.lib().cf_mc_supported(ctypes.byref(s)))
        mc = ctypes.c_void_p()
        rc = _lib.lib().cf_mc_create(4 << 20, 1, ctypes.byref(mc), None) if s.value else -1
        if rc == 0:
            _lib.lib().cf_mc_destroy(mc)
        _MC["ok"] = bool(s.value) and rc == 0
        _MC["why"] = ("multicast attribute 0" if not s.value else
                      f"cuMulticastCreate refused: {_lib.last_error()}" if rc != 0 else "")
    return _MC["ok"]


def test_multicast_support_reported():
    """cf_mc_supported answers and a one-device multicast object is attempted (the NVLS tests
    below need one; a box without an NVSwitch multicast team skips them with the reason)."""
    print("multicast usable:", _mc_supported(), _MC.get("why"))


@pytest.mark.parametrize("cones", [False, True])
def test_nvls_update_kernel_world1(cones):
    """cf_column_update_nvls on a one-device multicast object (multimem.ld_reduce of one copy,
    multimem.st into it) == cf_column_update on the partial, bit for bit, and the replica
    region of the multicast buffer receives x+."""
    import ctypes

    import torch

    from paper_2203_05027_b200 import _lib
    from paper_2203_05027_b200.sharded import _DevArray

    if not _mc_supported():
        pytest.skip("no multicast object on this box: " + _MC["why"])
    L = _lib.lib()
    n = 12_000
    g = torch.Generator(device="cuda")
    g.manual_seed(9)

    def rnd():
        return torch.randn(n, generator=g, device="cuda", dtype=torch.float64)

    a, c, x, z, d = rnd(), rnd(), rnd(), rnd(), rnd()
    cnt = torch.randint(0, 20, (n,), generator=g, device="cuda").double()
    cone_ptr = torch.arange(0, n + 1, 4, dtype=torch.int32, device="cuda") if cones else None
    nb = n // 4 if cones else 0

    def p(t):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    x1, z1, d1 = x.clone(), z.clone(), d.clone()
    _lib.check(L.cf_column_update(n, p(a), p(cnt), p(c), p(x1), p(z1), p(d1), 0.7, nb, p(cone_ptr), None))
    mc = ctypes.c_void_p()
    _lib.check(L.cf_mc_create(16 * n + 4096, 1, ctypes.byref(mc), None))
    try:
        _lib.check(L.cf_mc_add_device(mc))
        uc, mcp = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(L.cf_mc_bind(mc, ctypes.byref(uc), ctypes.byref(mcp)))
        part = torch.as_tensor(_DevArray(uc.value, n), device="cuda")
        rep = torch.as_tensor(_DevArray(uc.value + 8 * n + 256, n), device="cuda")
        part.copy_(a)
        torch.cuda.synchronize()
        x2, z2, d2 = x.clone(), z.clone(), d.clone()
        _lib.check(L.cf_column_update_nvls(n, ctypes.c_void_p(mcp.value), p(cnt), p(c), p(x2), p(z2), p(d2), 0.7, nb,
                                           p(cone_ptr), ctypes.c_void_p(mcp.value + 8 * n + 256), None))
        torch.cuda.synchronize()
        assert torch.equal(x1, x2) and torch.equal(z1, z2) and torch.equal(d1, d2)
        assert torch.equal(rep, x2)
        # the device barrier on the counter: one rank, target 1 then 2
        flag_uc, flag_mc = uc.value + 16 * n + 1024, mcp.value + 16 * n + 1024
        for t in (1, 2):
            _lib.check(L.cf_mc_barrier(ctypes.c_void_p(flag_mc), ctypes.c_void_p(flag_uc), t, None))
        torch.cuda.synchronize()
    finally:
        L.cf_mc_destroy(mc)


@pytest.mark.parametrize("kind", ["lp", "socp4"])
def test_sharded_nvls_step_equals_nccl_step(nccl_group, kind):
    """run_sharded(nvls=True) (switch reduction + multicast x store + device barrier; one
    rank) == the NCCL reduce-scatter + update + all-gather step, bit for bit."""
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device_shard
    from paper_2203_05027_b200.sharded import CudaRankBackend, run_sharded

    if not _mc_supported():
        pytest.skip("no multicast object on this box: " + _MC["why"])
    st = torch.cuda.current_stream()
    plan, rc, cc, cs, bn, cn, cones = generate_device_shard(20_000, 40_000, 5e-4, kind, 3, 0, 1,
                                                            stream=st.cuda_stream)
    cfg = SolverConfig(max_iters=60, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    out = []
    for nvls in (False, True):
        plan.set_state(1.0, None, export=False)
        be = CudaRankBackend.from_plan(plan, cc[0], cc[1], cs, cones)
        out.append(run_sharded(be, rc, cc, cfg, bn, cn, nvls=nvls))
        be.disable_nvls()
    assert np.array_equal(out[0].x, out[1].x) and np.array_equal(out[0].lam, out[1].lam)
    assert out[0].trace == out[1].trace
    plan.close()
