"""tcgen05 building blocks on hardware: one-CTA MMA through the exact shared-memory
layouts (K-major / MN-major SWIZZLE_128B), UMMA descriptors, TMA staging and TMEM
read-back (M = 64 and 128 layouts) that the attention kernels are built from."""

import itertools

import pytest
import torch

from paper_2602_13515_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(128, 64, 128), (128, 128, 64), (64, 64, 128), (128, 128, 128), (64, 128, 64)])
@pytest.mark.parametrize("a_mn,b_mn", list(itertools.product((0, 1), repeat=2)))
@pytest.mark.parametrize("use_tma", [0, 1])
def test_probe_gemm(m, n, k, a_mn, b_mn, use_tma):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k + a_mn * 11 + b_mn * 13 + use_tma)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    a_store = a.t().contiguous() if a_mn else a.contiguous()
    b_store = b.t().contiguous() if b_mn else b.contiguous()
    d = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float32)
    lib = _lib.load_diag()
    rc = lib.spa2_probe_gemm(_lib.ptr(a_store), _lib.ptr(b_store), _lib.ptr(d), m, n, k, a_mn, b_mn, use_tma,
                             torch.cuda.current_stream().cuda_stream)
    _lib.check_diag(rc, "probe")
    torch.cuda.synchronize()
    want = a.float() @ b.float().t()
    err = (d - want).abs().max().item()
    assert err <= 1e-3 * max(1.0, want.abs().max().item()), (m, n, k, a_mn, b_mn, use_tma, err)


@pytest.mark.parametrize("n,k", [(64, 128), (128, 128), (128, 64), (64, 64)])
def test_probe_tmem_cp_a_operand(n, k):
    """A staged K-major SWIZZLE_128B in smem, copied to TMEM with tcgen05.cp (128x256b per
    K=16 step), then consumed by TS MMAs — the Q/dO-in-TMEM layout of the fwd/dQ kernels."""
    g = torch.Generator(device="cuda").manual_seed(n + k)
    a = torch.randn(128, k, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16)
    d = torch.full((128, n), float("nan"), device="cuda", dtype=torch.float32)
    lib = _lib.load_diag()
    _lib.check_diag(lib.spa2_probe_gemm(_lib.ptr(a), _lib.ptr(b), _lib.ptr(d), 128, n, k, 0, 0, 3,
                                   torch.cuda.current_stream().cuda_stream), "probe")
    torch.cuda.synchronize()
    want = a.float() @ b.float().t()
    assert (d - want).abs().max().item() <= 1e-3 * max(1.0, want.abs().max().item())


def test_probe_rates_and_clock():
    """The rate probes behind DESIGN §5 / bench.py's on-chip roofline run and report sane
    numbers: an SS N=64 MMA step costs more than the 32-cycle datapath floor and a TS step
    holds it; the dK/dV MMA sequence costs at least its 4 x 8 x 32-cycle floor per tile; the
    SM clock probe reads a plausible clock."""
    lib = _lib.load_diag()
    st = torch.cuda.current_stream().cuda_stream
    ctas = 4
    src = torch.zeros(16 * 1024 * 1024 + 65536, dtype=torch.uint8, device="cuda")
    out = torch.zeros(ctas * 4, dtype=torch.int64, device="cuda")
    per = {}
    for mode in (0, 32, 1 | 2 | 4):
        _lib.check_diag(lib.spa2_probe_smem_contend(200, mode, ctas, _lib.ptr(src), _lib.ptr(out), st), "contend")
        torch.cuda.synchronize()
        per[mode] = out.view(ctas, 4)[:, 0].double().mean().item() / (200 * 8)
    assert 40.0 < per[0] < 70.0, per  # SS N=64: operand fetch above the datapath rate
    assert 28.0 < per[32] < 40.0, per  # TS N=64: at the 32-cycle floor
    assert per[1 | 2 | 4] < 1.2 * per[0], per  # other shared-memory traffic barely slows it
    cyc = torch.zeros(ctas, dtype=torch.int64, device="cuda")
    _lib.check_diag(lib.spa2_probe_dkdv_mix(100, 0, ctas, _lib.ptr(cyc), st), "dkdv_mix")
    torch.cuda.synchronize()
    per_tile = cyc.double().mean().item() / 100
    assert 1024 <= per_tile < 3000, per_tile
    clk = torch.zeros(2 * ctas, dtype=torch.int64, device="cuda")
    _lib.check_diag(lib.spa2_probe_clock(20000, ctas, _lib.ptr(clk), st), "clock")
    torch.cuda.synchronize()
    ghz = (clk.view(ctas, 2)[:, 0].double() / clk.view(ctas, 2)[:, 1].double()).median().item()
    assert 0.3 < ghz < 2.5, ghz
