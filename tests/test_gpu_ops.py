"""Operator-level parity on the GPU: WeightSlice conv (+ SubnetNorm epilogue,
residual, activation) through the C-ABI (ssn_op_conv_*), against the CPU
oracle (oracle/ssn_oracle.c:oracle_conv_op) on the same seeded tensors.

bf16 path: inputs and weights are bf16 values; the oracle computes in fp64
accumulation on those same values, so the only differences are the GPU's
fp32 accumulation order and the final bf16 rounding of the output
(tolerance: 1e-2 relative to the output scale, written per test).
"""
import numpy as np
import pytest

import paper_2312_16733_b200 as ssn
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _bf16(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)


def _run_bf16(gpu, n, h, w, cin, cin_max, cout, cout_max, k, stride, res=False, act=1,
              out_f32=False, seed=0):
    import torch
    rng = np.random.default_rng(seed)
    pad = k // 2
    x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
    wmax = (rng.standard_normal((cout_max, cin_max, k, k)) / np.sqrt(cin * k * k)).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32)
    shift = rng.uniform(-0.2, 0.2, cout).astype(np.float32)
    xb = _bf16(x)
    wb = _bf16(wmax)
    x_r = xb.float().numpy()
    w_r = wb.float().numpy()
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    r = rng.standard_normal((n, ho, wo, cout)).astype(np.float32) if res else None
    rb = _bf16(r) if res else None
    ref = O.conv_op(x_r, w_r, cout_max, cin_max, k, k, stride, pad, cout, scale=scale,
                    shift=shift, res=None if rb is None else rb.float().numpy(), act=act)
    # device tensors: x NHWC compact, weights KRSC max shape
    xd = xb.to(gpu).contiguous()
    wd = wb.permute(0, 2, 3, 1).contiguous().to(gpu)  # [cout][k][k][cin_max]
    sd = torch.from_numpy(scale).to(gpu)
    hd = torch.from_numpy(shift).to(gpu)
    rd = rb.to(gpu).contiguous() if res else None
    y = torch.empty((n, ho, wo, cout), dtype=torch.float32 if out_f32 else torch.bfloat16,
                    device=gpu)
    ssn.op_conv_bf16(xd, n, h, w, cin, wd, cout_max, cin_max, k, stride, pad, cout, sd, hd, rd,
                     act, int(out_f32), y)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy()
    return got, ref


CASES = [
    # n, h, w, cin, cin_max, cout, cout_max, k, stride
    (1, 8, 8, 64, 64, 64, 64, 1, 1),        # single tile, one k-block
    (2, 16, 16, 128, 128, 128, 128, 1, 1),  # M = 512, 2 k-blocks
    (2, 14, 14, 88, 128, 96, 128, 1, 1),    # channel slices (K tail, N tail)
    (3, 9, 11, 40, 64, 24, 32, 3, 1),       # 3x3 pad 1, odd spatial, M tail
    (2, 16, 16, 64, 64, 128, 256, 3, 2),    # 3x3 stride 2
    (1, 7, 7, 360, 360, 200, 360, 3, 1),    # many k-blocks, cout slice
    (4, 28, 28, 256, 256, 512, 512, 1, 1),  # bn 256 path (large)
    (2, 10, 10, 8, 8, 32, 32, 3, 2),        # stem-like cin = 8
    (64, 1, 1, 2048, 2048, 1000, 1000, 1, 1),  # classifier GEMM
    # packed-tap K blocks (cin_a <= 32, full kernel): cslot 16 / 32 with a channel gap
    (4, 16, 16, 16, 16, 32, 32, 3, 1),
    (2, 20, 20, 24, 32, 32, 64, 3, 2),
    (3, 15, 15, 32, 32, 40, 48, 3, 1),
    # persistent schedule: more tiles than SMs, several n tiles
    (64, 28, 28, 128, 128, 128, 128, 1, 1),
    (8, 14, 14, 256, 256, 1024, 1024, 1, 1),
    (16, 14, 14, 104, 128, 360, 360, 3, 1),
    # shifted-window (halo) kernel: stride-1 3x3 with resident weights
    (2, 56, 56, 88, 88, 88, 88, 3, 1),      # OFA-R50 stage-1 max
    (2, 56, 56, 56, 88, 56, 88, 3, 1),      # WeightSlice of the max tensor
    (1, 112, 112, 24, 32, 40, 64, 3, 1),    # stem 112 px (one window row-tile per row)
    (3, 28, 28, 40, 64, 48, 64, 3, 1),      # cin16 = 48: a half channel block
    (2, 20, 30, 16, 16, 16, 16, 3, 1),      # h != w, 4 rows per tile
    (5, 17, 19, 32, 32, 64, 64, 3, 1),      # odd sizes, last tile past H
    # shifted-window PAIR kernel (conv_hp.cu): wide stride-1 3x3 at 14-62 px
    (2, 14, 14, 360, 360, 360, 360, 3, 1),  # OFA-R50 stage-3 max (2 N tiles of 192/168)
    (3, 14, 14, 208, 360, 208, 360, 3, 1),  # WeightSlice of the max tensor, odd CTA-tile count
    (1, 28, 28, 176, 176, 176, 176, 3, 1),  # 7 CTA tiles: idle half in the last pair
    (2, 28, 28, 104, 176, 104, 176, 3, 1),  # mid-subnet stage 2
    (5, 14, 14, 136, 360, 136, 360, 3, 1),  # min-subnet stage 3, ragged K block
    (2, 20, 30, 144, 144, 160, 160, 3, 1),  # h != w (Wp 32, 4 rows per CTA tile)
    (1, 14, 14, 40, 360, 360, 360, 3, 1),   # one partial channel block
    (2, 14, 14, 360, 360, 512, 512, 3, 1),  # 2 full 256-wide N tiles
]


@pytest.mark.parametrize("case", CASES)
def test_conv_bf16_matches_oracle(gpu, case):
    n, h, w, cin, cin_max, cout, cout_max, k, stride = case
    got, ref = _run_bf16(gpu, n, h, w, cin, cin_max, cout, cout_max, k, stride)
    err = np.abs(got - ref).max() / (np.abs(ref).max() + 1e-6)
    assert err < 1e-2, f"max rel err {err}"


def test_conv_bf16_halo_residual(gpu):
    """The stem residual block (y + relu(bn(conv3x3(y)))) on the halo kernel."""
    got, ref = _run_bf16(gpu, 2, 56, 56, 32, 32, 32, 32, 3, 1, res=True, act=1)
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-2


def test_conv_bf16_residual_and_f32_out(gpu):
    got, ref = _run_bf16(gpu, 2, 12, 12, 64, 64, 64, 64, 1, 1, res=True, act=1)
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-2
    got, ref = _run_bf16(gpu, 8, 1, 1, 256, 512, 1000, 1000, 1, 1, act=0, out_f32=True)
    assert np.abs(got - ref).max() / np.abs(ref).max() < 5e-3


@pytest.mark.parametrize("cin", [192, 208, 256])
def test_conv_bf16_resident_slice_narrower_than_instance(gpu, cin):
    """Resident-B 1x1 with bn (176) < the instance's BN_MAX (256), four K
    blocks and several tiles per CTA: the resident slice is packed at the
    actual tile width.  (A BN_MAX block stride once overran the 96 KB region
    into the epilogue's staging tile — wrong, run-to-run varying results.)
    Checked against the oracle for several active widths."""
    for cout in (104, 176):
        got, ref = _run_bf16(gpu, 32, 28, 28, cin, 256, cout, 176, 1, 1, act=1)  # 196 tiles
        err = np.abs(got - ref).max() / (np.abs(ref).max() + 1e-6)
        assert err < 1e-2, (cin, cout, err)


@pytest.mark.parametrize("cout", [2, 10, 13])
def test_conv_bf16_ragged_cout(gpu, cout):
    """cout % 8 != 0 (e.g. a 2-label classifier) takes the scalar epilogue tail."""
    got, ref = _run_bf16(gpu, 16, 1, 1, 768, 768, cout, 16, 1, 1, act=0, out_f32=True)
    assert np.abs(got - ref).max() / np.abs(ref).max() < 5e-3
    got, ref = _run_bf16(gpu, 2, 6, 6, 64, 64, cout, 16, 3, 1, res=True, act=1)
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-2


def test_conv_bf16_rejects_bad_slices(gpu):
    import torch
    x = torch.zeros(64, device=gpu, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        ssn.op_conv_bf16(x, 1, 1, 1, 12, x, 16, 16, 1, 1, 0, 16, y=x)  # cin % 8
    with pytest.raises(ValueError):
        ssn.op_conv_bf16(x, 1, 1, 1, 32, x, 16, 16, 1, 1, 0, 16, y=x)  # cin > cin_max


@pytest.mark.parametrize("depthwise", [False, True])
def test_conv_f32_matches_oracle(gpu, depthwise):
    import torch
    rng = np.random.default_rng(3)
    n, h, w = 2, 9, 9
    cin_max, cout_max, k_max = 24, 24, 5
    cin, cout, k, stride = (16, 16, 3, 2) if depthwise else (12, 20, 3, 1)
    x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
    wshape = (cout_max, 1, k_max, k_max) if depthwise else (cout_max, cin_max, k_max, k_max)
    wmax = rng.standard_normal(wshape).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, cout).astype(np.float32)
    shift = rng.uniform(-0.2, 0.2, cout).astype(np.float32)
    pad = k // 2
    ref = O.conv_op(x, wmax, cout_max, cin_max, k_max, k, stride, pad, cout, depthwise=depthwise,
                    scale=scale, shift=shift, act=1)
    wk = torch.from_numpy(wmax).permute(0, 2, 3, 1).contiguous().to(gpu)  # KRSC
    y = torch.empty(ref.shape, dtype=torch.float32, device=gpu)
    ssn.op_conv_f32(torch.from_numpy(x).to(gpu), n, h, w, cin, wk, cout_max, cin_max, k_max, k,
                    stride, pad, cout, int(depthwise), torch.from_numpy(scale).to(gpu),
                    torch.from_numpy(shift).to(gpu), None, 1, y)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-4)


# ---- depthwise bf16 (dw.cu: TMA-pipelined, elastic centre crop) ----------
DW_CASES = [
    # n, h, w, c, c_max, k_max, k, stride, act
    (2, 14, 14, 64, 64, 7, 7, 1, 1),      # one chunk, full kernel
    (2, 14, 14, 64, 64, 7, 3, 1, 2),      # centre crop 3 of 7, h_swish
    (2, 28, 28, 144, 192, 7, 5, 1, 1),    # ragged chunk (144 = 2x64 + 16), 5 of 7
    (3, 7, 7, 1152, 1152, 7, 7, 1, 2),    # 7 px tiles, many chunks
    (2, 56, 56, 72, 144, 7, 3, 2, 1),     # stride 2, ragged 72
    (2, 112, 112, 24, 24, 3, 3, 1, 1),    # c < 64 (box wider than the tensor)
    (1, 13, 17, 40, 48, 5, 5, 2, 0),      # odd sizes, stride 2, no activation
    (2, 9, 11, 32, 32, 7, 7, 1, 1),       # width not a multiple of 7, single chunk
    (16, 14, 14, 816, 816, 7, 7, 2, 2),   # 14 -> 7 stride 2
    # narrow layers (c_max <= 32): 32-channel boxes, two pixels per warp
    (3, 30, 30, 16, 32, 7, 5, 1, 2),      # WeightSlice c < c_max, 5 of 7, h_swish
    (2, 20, 9, 32, 32, 5, 5, 1, 0),       # odd width > 7 (half-empty second lane half)
    (1, 15, 28, 8, 24, 3, 3, 1, 1),       # 8 of 24 channels
]


def _run_dw(gpu, n, h, w, c, c_max, k_max, k, stride, act, seed=0):
    import torch
    rng = np.random.default_rng(seed)
    pad = k // 2
    x = rng.standard_normal((n, h, w, c)).astype(np.float32)
    wmax = (rng.standard_normal((c_max, 1, k_max, k_max)) / k).astype(np.float32)
    scale = rng.uniform(0.5, 1.5, c).astype(np.float32)
    shift = rng.uniform(-0.2, 0.2, c).astype(np.float32)
    xb, wb = _bf16(x), _bf16(wmax)
    ref = O.conv_op(xb.float().numpy(), wb.float().numpy(), c_max, c_max, k_max, k, stride, pad,
                    c, depthwise=True, scale=scale, shift=shift, act=act)
    wd = wb[:, 0].permute(1, 2, 0).contiguous().to(gpu)  # tap-major [k_max][k_max][c_max]
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    y = torch.full((n, ho, wo, c), float("nan"), dtype=torch.bfloat16, device=gpu)
    ssn.op_dw_bf16(xb.to(gpu).contiguous(), n, h, w, c, wd, c_max, k_max, k, stride,
                   torch.from_numpy(scale).to(gpu), torch.from_numpy(shift).to(gpu), act, y)
    torch.cuda.synchronize()
    return y.float().cpu().numpy(), ref


@pytest.mark.parametrize("case", DW_CASES, ids=[str(c) for c in DW_CASES])
def test_dw_bf16_matches_oracle(gpu, case):
    got, ref = _run_dw(gpu, *case)
    assert np.isfinite(got).all(), "unwritten outputs (NaN sentinel survived)"
    scale = max(1.0, float(np.abs(ref).max()))
    # fp32 accumulation of bf16 products, one bf16 rounding of the output
    assert np.abs(got - ref).max() <= 1e-2 * scale


def test_dw_bf16_rejects_bad_args(gpu):
    import torch
    x = torch.zeros(4096, device=gpu, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        ssn.op_dw_bf16(x, 1, 4, 4, 12, x, 16, 7, 3, 1, y=x)   # c % 8
    with pytest.raises(ValueError):
        ssn.op_dw_bf16(x, 1, 4, 4, 16, x, 16, 7, 9, 1, y=x)   # k > k_max
    with pytest.raises(ValueError):
        ssn.op_dw_bf16(x, 1, 4, 4, 16, x, 16, 7, 3, 3, y=x)   # stride 3
