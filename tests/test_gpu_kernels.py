"""Kernel-level numerics on the device, each against a plain PyTorch fp32
reference of the same op (and the oracle for the weight streams)."""

import ctypes as C
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_02921_b200 import _lib  # noqa: E402


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.manual_seed(0)


def test_library_loads_on_device():
    assert _lib.lib().krr_version().startswith(b"kvrerank_b200")


@pytest.mark.parametrize("code,tdt", [(_lib.F32, torch.float32), (_lib.F16, torch.float16)])
def test_init_uniform_matches_oracle(code, tdt):
    import oracle
    rows, cols = 96, 160
    seed = 0 ^ oracle.fnv1a64("layers.0.attn.wq")
    bound = math.sqrt(6.0 / (rows + cols))
    ref = oracle.uniform_signed(seed, rows * cols, bound).reshape(rows, cols)
    out = torch.empty((cols, rows), dtype=tdt, device="cuda")   # transposed [out, in]
    _lib.check(_lib.lib().krr_init_uniform(seed, bound, rows, cols, 1, code, out.data_ptr(),
                                           rows, _stream()))
    got = out.float().cpu().numpy().T
    want = ref.astype(np.float16).astype(np.float32) if code == _lib.F16 else ref
    assert np.array_equal(got, want)


def _gemm(backend, act, A, B, epi, out, qkv=None):
    _lib.check(_lib.lib().krr_gemm(backend, act, A.data_ptr(), B.data_ptr(), A.shape[0],
                                   B.shape[0], A.shape[1], epi,
                                   out.data_ptr() if out is not None else 0,
                                   C.byref(qkv) if qkv is not None else None, _stream()))


GEMM_SHAPES = [(128, 256, 64), (300, 512, 256), (1000, 1024, 512), (77, 96, 128),
               (2048, 4096, 1024),
               (4800, 2048, 256), (384, 4096, 128)]    # wave model picks 192 / 128-wide tiles


@pytest.mark.parametrize("backend", [_lib.GEMM_TCGEN05, _lib.GEMM_SIMT])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_store_gelu_residual(backend, M, N, K):
    A = (torch.randn(M, K, device="cuda") * 0.5).half()
    B = (torch.randn(N, K, device="cuda") * (1.0 / math.sqrt(K))).half()
    ref = A.float() @ B.float().T
    out = torch.empty(M, N, dtype=torch.float16, device="cuda")
    _gemm(backend, _lib.F16, A, B, _lib.EPI_STORE, out)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    assert err <= 2e-3 * max(1.0, ref.abs().max().item()), err
    _gemm(backend, _lib.F16, A, B, _lib.EPI_GELU, out)
    g = torch.nn.functional.gelu(ref, approximate="tanh")
    torch.cuda.synchronize()
    assert (out.float() - g).abs().max().item() <= 2e-3 * max(1.0, g.abs().max().item())
    x = torch.randn(M, N, device="cuda")
    x0 = x.clone()
    _gemm(backend, _lib.F16, A, B, _lib.EPI_RESIDUAL, x)
    torch.cuda.synchronize()
    assert (x - (x0 + ref)).abs().max().item() <= 1e-3 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("backend", [_lib.GEMM_TCGEN05, _lib.GEMM_SIMT])
@pytest.mark.parametrize("epi", [_lib.EPI_GLU_GELU, _lib.EPI_GLU_SILU])
@pytest.mark.parametrize("M,F,K", [(300, 256, 256), (77, 96, 128), (2048, 1024, 512)])
def test_gemm_gated_mlp_epilogue(backend, epi, M, F, K):
    """Gated-MLP epilogue (f4 variants): B interleaves 32-row gate / up blocks;
    out[M, F] = act(A Wg^T) * (A Wu^T), act = tanh-GELU or SiLU."""
    A = (torch.randn(M, K, device="cuda") * 0.5).half()
    Wg = (torch.randn(F, K, device="cuda") * (1.0 / math.sqrt(K))).half()
    Wu = (torch.randn(F, K, device="cuda") * (1.0 / math.sqrt(K))).half()
    B = torch.stack([Wg.view(F // 32, 32, K), Wu.view(F // 32, 32, K)], 1).reshape(2 * F, K)
    g, u = A.float() @ Wg.float().T, A.float() @ Wu.float().T
    act = (torch.nn.functional.gelu(g, approximate="tanh") if epi == _lib.EPI_GLU_GELU
           else torch.nn.functional.silu(g))
    ref = act * u
    out = torch.empty(M, F, dtype=torch.float16, device="cuda")
    _gemm(backend, _lib.F16, A, B.contiguous(), epi, out)
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    assert err <= 4e-3 * max(1.0, ref.abs().max().item()), err


def test_gemm_f32_simt_exact_order():
    M, N, K = 200, 128, 96
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    out = torch.empty(M, N, device="cuda")
    _gemm(_lib.GEMM_SIMT, _lib.F32, A, B, _lib.EPI_STORE, out)
    ref = (A.double() @ B.double().T).float()
    torch.cuda.synchronize()
    assert (out - ref).abs().max().item() < 1e-4


def test_gemm_batch_invariance_tcgen05():
    """A row's result must not depend on M (no split-K): SPEC.md:178."""
    K, N = 512, 768
    A = (torch.randn(1000, K, device="cuda") * 0.5).half()
    B = (torch.randn(N, K, device="cuda") * 0.05).half()
    full = torch.empty(1000, N, dtype=torch.float16, device="cuda")
    _gemm(_lib.GEMM_TCGEN05, _lib.F16, A, B, _lib.EPI_STORE, full)
    part = torch.empty(333, N, dtype=torch.float16, device="cuda")
    _gemm(_lib.GEMM_TCGEN05, _lib.F16, A[500:833].contiguous(), B, _lib.EPI_STORE, part)
    torch.cuda.synchronize()
    assert torch.equal(full[500:833], part)


@pytest.mark.parametrize("epi", [_lib.EPI_STORE, _lib.EPI_GELU])
def test_gemm_batch_invariance_across_tile_widths(epi):
    """Small batches run narrower N tiles (and no cluster); the per-element MMA
    sequence is unchanged, so a row's bits must not change with M."""
    K, N, M = 1024, 2048, 20000            # full: 256-wide tiles; parts: 64 / 128 / 224 / 192
    A = (torch.randn(M, K, device="cuda") * 0.5).half()
    B = (torch.randn(N, K, device="cuda") * 0.03).half()
    full = torch.empty(M, N, dtype=torch.float16, device="cuda")
    _gemm(_lib.GEMM_TCGEN05, _lib.F16, A, B, epi, full)
    for r0, m in ((4096, 96), (777, 700), (0, 2500), (5000, 4800)):
        part = torch.empty(m, N, dtype=torch.float16, device="cuda")
        _gemm(_lib.GEMM_TCGEN05, _lib.F16, A[r0:r0 + m].contiguous(), B, epi, part)
        torch.cuda.synchronize()
        assert torch.equal(full[r0:r0 + m], part), (r0, m)


def _rope_ref(x, pos, cos, sin):
    # x [..., HD] rotated as complex pairs (model.py:144,370-371)
    a, b = x[..., 0::2], x[..., 1::2]
    c, s = cos[pos], sin[pos]
    out = torch.empty_like(x)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


@pytest.mark.parametrize("backend", [_lib.GEMM_TCGEN05, _lib.GEMM_SIMT])
def test_gemm_qkv_rope_scatter(backend):
    from paper_2504_02921_b200.model import rope_tables
    H, KVH, HD, T, nseq, L, layer = 4, 2, 64, 48, 3, 2, 1
    d = H * HD
    G = H // KVH
    M = nseq * T
    N = (H + 2 * KVH) * HD
    pos0 = 128
    cos, sin = rope_tables(10000.0, HD, 1024)
    cos_t, sin_t = torch.from_numpy(cos).cuda(), torch.from_numpy(sin).cuda()
    A = (torch.randn(M, d, device="cuda")).half()
    B = (torch.randn(N, d, device="cuda") / 16).half()
    ref = A.float() @ B.float().T
    q_out = torch.zeros(nseq * KVH * G * T * HD, dtype=torch.float16, device="cuda")
    slabs = torch.zeros(nseq, L, 2, KVH, T, HD, dtype=torch.float16, device="cuda")
    ptrs = torch.arange(nseq, device="cuda", dtype=torch.int64) * (slabs[0].numel() * 2) + \
        slabs.data_ptr()
    qkv = _lib.QKV(H, KVH, HD, T, pos0, layer, T, cos_t.data_ptr(), sin_t.data_ptr(),
                   q_out.data_ptr(), ptrs.data_ptr())
    _gemm(backend, _lib.F16, A, B, _lib.EPI_QKV_ROPE, None, qkv)
    torch.cuda.synchronize()
    pos = torch.arange(T, device="cuda") + pos0
    r = ref.view(nseq, T, H + 2 * KVH, HD)
    q = _rope_ref(r[:, :, :H], pos[None, :, None].expand(nseq, T, H), cos_t, sin_t)
    k = _rope_ref(r[:, :, H:H + KVH], pos[None, :, None].expand(nseq, T, KVH), cos_t, sin_t)
    v = r[:, :, H + KVH:]
    q_want = q.view(nseq, T, KVH, G, HD).permute(0, 2, 3, 1, 4).reshape(-1)
    assert (q_out.float() - q_want).abs().max().item() < 2e-2
    assert (slabs[:, layer, 0].float() - k.permute(0, 2, 1, 3)).abs().max().item() < 2e-2
    assert (slabs[:, layer, 1].float() - v.permute(0, 2, 1, 3)).abs().max().item() < 2e-2
    assert slabs[:, 1 - layer].abs().max().item() == 0


@pytest.mark.parametrize("epi", [_lib.EPI_STORE, _lib.EPI_GELU, _lib.EPI_RESIDUAL])
def test_gemm_pair_geometry_bit_identical(epi):
    """Launches of 16k-131k rows run the CTA-pair geometry (G=8: cta_group::2,
    256 rows per SM, accumulator halves handed over separately); smaller ones the
    cluster-multicast G=3.  Same per-element MMA sequence: the rows of a ragged
    M=16,684 launch equal the same rows computed by small launches bit for bit,
    and match fp32 torch."""
    M, N, K = 16384 + 300, 768, 1024
    A = (torch.randn(M, K, device="cuda") * 0.5).half()
    B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).half()
    if epi == _lib.EPI_RESIDUAL:
        x0 = torch.randn(M, N, device="cuda")
        full = x0.clone()
    else:
        full = torch.empty(M, N, dtype=torch.float16, device="cuda")
    _gemm(_lib.GEMM_TCGEN05, _lib.F16, A, B, epi, full)
    for r0, m in ((0, 4096), (M - 3000, 3000), (9000, 511)):
        part = x0[r0:r0 + m].clone() if epi == _lib.EPI_RESIDUAL else \
            torch.empty(m, N, dtype=torch.float16, device="cuda")
        _gemm(_lib.GEMM_TCGEN05, _lib.F16, A[r0:r0 + m].contiguous(), B, epi, part)
        torch.cuda.synchronize()
        assert torch.equal(full[r0:r0 + m], part), (r0, m)
    ref = A.float() @ B.float().T
    if epi == _lib.EPI_GELU:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    if epi == _lib.EPI_RESIDUAL:
        ref = x0 + ref
    assert (full.float() - ref).abs().max().item() <= 2e-3 * max(1.0, ref.abs().max().item())


def test_gemm_pair_geometry_qkv_scatter():
    """The QKV RoPE scatter through the pair geometry (400 sequences x 48 rows =
    19,200 rows) equals the same sequences scattered by two small launches."""
    from paper_2504_02921_b200.model import rope_tables
    H, KVH, HD, T, nseq, L, layer = 8, 2, 128, 48, 400, 2, 1
    d, G, N = H * HD, H // KVH, (H + 2 * KVH) * HD
    cos, sin = rope_tables(10000.0, HD, 1024)
    cos_t, sin_t = torch.from_numpy(cos).cuda(), torch.from_numpy(sin).cuda()
    A = torch.randn(nseq * T, d, device="cuda").half()
    B = (torch.randn(N, d, device="cuda") / 16).half()

    def run(a, n):
        q_out = torch.zeros(n * KVH * G * T * HD, dtype=torch.float16, device="cuda")
        slabs = torch.zeros(n, L, 2, KVH, T, HD, dtype=torch.float16, device="cuda")
        ptrs = torch.arange(n, device="cuda", dtype=torch.int64) * (slabs[0].numel() * 2) + \
            slabs.data_ptr()
        qkv = _lib.QKV(H, KVH, HD, T, 512, layer, T, cos_t.data_ptr(), sin_t.data_ptr(),
                       q_out.data_ptr(), ptrs.data_ptr())
        _gemm(_lib.GEMM_TCGEN05, _lib.F16, a.contiguous(), B, _lib.EPI_QKV_ROPE, None, qkv)
        torch.cuda.synchronize()
        return q_out.view(n, -1), slabs
    q_full, s_full = run(A, nseq)
    h = nseq // 2
    for i0 in (0, h):
        q_p, s_p = run(A[i0 * T:(i0 + h) * T], h)
        assert torch.equal(q_full[i0:i0 + h], q_p) and torch.equal(s_full[i0:i0 + h], s_p)


def _attn_ref(q, kp, vp, vlen, kc, vc, tv, G, T):
    """fp32 torch restatement of model.py:373-394 for one (seq, kv head)."""
    P = kp.shape[0]
    logits_p = q @ kp.T
    logits_c = q @ kc.T
    t = torch.arange(G * T, device=q.device) % T
    pm = torch.arange(P, device=q.device)[None, :] < vlen
    cm = (torch.arange(T, device=q.device)[None, :] <= t[:, None]) & tv[None, :].bool()
    logits_p = logits_p.masked_fill(~pm, float("-inf"))
    logits_c = logits_c.masked_fill(~cm, float("-inf"))
    lg = torch.cat([logits_p, logits_c], dim=1)
    m = lg.max(dim=1, keepdim=True).values
    m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    e = torch.exp(lg - m)
    z = e.sum(dim=1, keepdim=True)
    z = torch.where(z == 0, torch.ones_like(z), z)
    return (e @ torch.cat([vp, vc], dim=0)) / z


ATTN_CASES = [(64, 2, 2, 128, 48, 1.0), (128, 4, 2, 512, 48, 1.0), (256, 8, 1, 512, 48, 1.0),
              (256, 8, 1, 512, 48, 8.0), (256, 8, 1, 0, 64, 2.0),
              (64, 2, 2, 0, 128, 1.0), (128, 4, 2, 0, 100, 1.0), (128, 4, 2, 512, 48, 8.0),
              (128, 4, 2, 2048, 16, 8.0), (128, 4, 2, 0, 512, 4.0), (64, 2, 2, 200, 48, 4.0)]


@pytest.mark.parametrize("HD,G,KVH,P,T,boost", ATTN_CASES)
@pytest.mark.parametrize("backend,act", [(_lib.ATTN_MMA, _lib.F16), (_lib.ATTN_SIMT, _lib.F32),
                                         (_lib.ATTN_MMA, _lib.BF16),
                                         (_lib.ATTN_TCGEN05, _lib.F16),
                                         (_lib.ATTN_TCGEN05, _lib.BF16)])
def test_attention(HD, G, KVH, P, T, boost, backend, act):
    """``boost`` scales q so logits reach the magnitudes of the unscaled model
    (std ~ sqrt(HD)), which exercises the lazy-rescale path of the tcgen05 kernel."""
    nseq, L, layer = 3, 2, 1
    tdt = {_lib.F16: torch.float16, _lib.F32: torch.float32, _lib.BF16: torch.bfloat16}[act]
    sc = 1.0 / math.sqrt(math.sqrt(HD))
    q = (torch.randn(nseq * KVH, G * T, HD, device="cuda") * sc * boost).to(tdt)
    pre = (torch.randn(nseq, L, 2, KVH, max(P, 1), HD, device="cuda") * sc).to(tdt)
    cur = (torch.randn(nseq, 1, 2, KVH, T, HD, device="cuda") * sc).to(tdt)
    vlen = torch.tensor([P, max(1, P // 3), max(1, P - 7)][:nseq], dtype=torch.int32,
                        device="cuda")
    tv = torch.ones(nseq, T, dtype=torch.uint8, device="cuda")
    tv[1, T - 5:] = 0
    tv[2, 3] = 0
    tv[2, 10] = 0
    if P == 0:
        tv[0, 0] = 0          # row t=0 of seq 0 sees no key at all -> zeros
    es = pre.element_size()
    pptr = torch.arange(nseq, device="cuda", dtype=torch.int64) * (pre[0].numel() * es) + \
        pre.data_ptr()
    cptr = torch.arange(nseq, device="cuda", dtype=torch.int64) * (cur[0].numel() * es) + \
        cur.data_ptr()
    H = KVH * G
    out = torch.zeros(nseq * T, H * HD, dtype=tdt, device="cuda")
    _lib.check(_lib.lib().krr_attention(backend, act, q.data_ptr(), nseq, KVH, G, HD, T, P,
                                        layer, 0, pptr.data_ptr(), vlen.data_ptr(),
                                        cptr.data_ptr(), tv.data_ptr(), out.data_ptr(),
                                        pre.data_ptr(), pre.numel() * es, cur.data_ptr(),
                                        cur.numel() * es, _stream()))
    torch.cuda.synchronize()
    tol = {_lib.F16: 2e-2, _lib.BF16: 6e-2, _lib.F32: 1e-4}[act]
    for b in range(nseq):
        for kh in range(KVH):
            kp = pre[b, layer, 0, kh, :P].float()
            vp = pre[b, layer, 1, kh, :P].float()
            ref = _attn_ref(q[b * KVH + kh].float(), kp, vp, int(vlen[b]) if P else 0,
                            cur[b, 0, 0, kh].float(), cur[b, 0, 1, kh].float(), tv[b], G, T)
            got = out.view(nseq, T, KVH, G, HD)[b, :, kh].permute(1, 0, 2).reshape(G * T, HD)
            assert torch.isfinite(got.float()).all()
            err = (got.float() - ref).abs().max().item()
            assert err <= tol * max(1.0, ref.abs().max().item()), (b, kh, err)


def test_attention_tcgen05_occupancy_query():
    """krr_attention_occupancy answers for the tcgen05 attention (the
    persistent default kernel is one 320-thread CTA per SM, 197 KB of smem)."""
    from paper_2504_02921_b200 import _lib as L
    n = C.c_int32()
    _lib.check(L.lib().krr_attention_occupancy(_lib.F16, 128, C.byref(n)))
    assert n.value >= 1, n.value


@pytest.mark.parametrize("seg,k", [(100, 20), (7, 20), (2048, 20), (3000, 50), (6145, 20),
                                   (16384, 100)])
def test_segmented_topk(seg, k):
    """Rank-by-counting (<= 2048) and the bitonic path (longer segments, which
    need the smem opt-in): order by (score desc, doc id asc, index asc)."""
    n_seg = 3
    g = torch.Generator(device="cuda").manual_seed(seg)
    s = torch.randn(n_seg, seg, device="cuda", generator=g)
    s[0, :5] = 5.0                          # ties broken by doc id
    s[1, :] = torch.round(s[1, :] * 4) / 4  # many ties
    s[2, -1] = 0.0
    s[2, 0] = -0.0
    ids = torch.stack([torch.randperm(4 * seg, device="cuda", generator=g)[:seg]
                       for _ in range(n_seg)]).int()
    ids[1, :seg // 2] = ids[1, seg // 2:2 * (seg // 2)]   # duplicate ids: index breaks ties
    idx = torch.empty(n_seg, k, dtype=torch.int32, device="cuda")
    sc = torch.empty(n_seg, k, device="cuda")
    _lib.check(_lib.lib().krr_segmented_topk(s.data_ptr(), ids.data_ptr(), n_seg, seg, k,
                                             idx.data_ptr(), sc.data_ptr(), _stream()))
    torch.cuda.synchronize()
    s_h, ids_h = s.cpu().numpy(), ids.cpu().numpy()
    for i in range(n_seg):
        order = np.lexsort((np.arange(seg), ids_h[i], -s_h[i].astype(np.float64)))[:k].tolist()
        want = order + [-1] * (k - len(order))
        assert idx[i].cpu().tolist() == want
        got = sc[i].cpu().numpy()
        assert np.array_equal(got[:len(order)], s_h[i][order])
        assert np.all(np.isneginf(got[len(order):]))


@pytest.mark.parametrize("d", [128, 256, 2048, 4096, 200])
@pytest.mark.parametrize("code,tdt", [(_lib.F32, torch.float32), (_lib.F16, torch.float16)])
def test_rmsnorm(d, code, tdt):
    x = torch.randn(37, d, device="cuda") * 3
    g = torch.rand(d, device="cuda") + 0.5
    out = torch.empty(37, d, dtype=tdt, device="cuda")
    _lib.check(_lib.lib().krr_rmsnorm(x.data_ptr(), g.data_ptr(), 37, d, code, out.data_ptr(),
                                      _stream()))
    ref = x * (1.0 / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-6)) * g
    torch.cuda.synchronize()
    tol = 1e-5 if code == _lib.F32 else 2e-3
    assert (out.float() - ref).abs().max().item() <= tol * ref.abs().max().item()


@pytest.mark.parametrize("HD,G,KVH,P,T", [(128, 4, 2, 512, 48), (128, 4, 2, 200, 16),
                                          (64, 2, 2, 128, 48), (128, 4, 8, 2048, 256)])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("act", [_lib.F16, _lib.BF16])
def test_attention_quant_prefix_matches_expanded(HD, G, KVH, P, T, bits, act):
    """INT8/INT4 prefix pages dequantised inside the attention
    kernel (krr_attention_quant) match expanding the pages into HBM first
    (krr_dequant_pages, codec.py:82-95) and attending over 16-bit pages: bit for
    bit with bf16 activations (same f32 product, one rounding); with f16 the
    in-kernel decode multiplies by f16-rounded scales (<= 2^-11 relative per
    element), so outputs agree to f16 attention precision.  The expansion itself
    equals the reference codec's decode."""
    nseq, L, layer = 3, 2, 1
    tdt = torch.float16 if act == _lib.F16 else torch.bfloat16
    sc = 1.0 / math.sqrt(math.sqrt(HD))
    q = (torch.randn(nseq * KVH, G * T, HD, device="cuda") * sc * 4).to(tdt)
    pre32 = torch.randn(nseq, L, 2, KVH, P, HD, device="cuda") * sc
    pre32[0, layer, 1, 0, :, 5] = 0.0                   # an all-zero channel (scale 1.0)
    cur = (torch.randn(nseq, 1, 2, KVH, T, HD, device="cuda") * sc).to(tdt)
    n_t = nseq * L * 2
    tb = KVH * P * HD if bits == 8 else KVH * P * HD // 2
    codes = torch.empty(n_t * tb, dtype=torch.uint8, device="cuda")
    scales = torch.empty(n_t * KVH * HD, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().krr_quant_pages(pre32.data_ptr(), _lib.F32, n_t, KVH, P, HD, bits,
                                          codes.data_ptr(), scales.data_ptr(), _stream()))
    pre = torch.empty(nseq, L, 2, KVH, P, HD, dtype=tdt, device="cuda")
    _lib.check(_lib.lib().krr_dequant_pages(codes.data_ptr(), scales.data_ptr(), bits, n_t, KVH,
                                            P, HD, act, pre.data_ptr(), _stream()))
    vlen = torch.tensor([P, max(1, P // 3), max(1, P - 7)], dtype=torch.int32, device="cuda")
    tv = torch.ones(nseq, T, dtype=torch.uint8, device="cuda")
    tv[1, T - 5:] = 0
    tv[2, 3] = 0
    es = pre.element_size()
    pptr = torch.arange(nseq, device="cuda", dtype=torch.int64) * (pre[0].numel() * es) + \
        pre.data_ptr()
    cptr = torch.arange(nseq, device="cuda", dtype=torch.int64) * (cur[0].numel() * es) + \
        cur.data_ptr()
    qptr = torch.arange(nseq, device="cuda", dtype=torch.int64) * (L * 2 * tb) + codes.data_ptr()
    H = KVH * G
    out_ref = torch.zeros(nseq * T, H * HD, dtype=tdt, device="cuda")
    out_q = torch.full_like(out_ref, float("nan"))
    _lib.check(_lib.lib().krr_attention(_lib.ATTN_TCGEN05, act, q.data_ptr(), nseq, KVH, G, HD,
                                        T, P, layer, 0, pptr.data_ptr(), vlen.data_ptr(),
                                        cptr.data_ptr(), tv.data_ptr(), out_ref.data_ptr(),
                                        pre.data_ptr(), pre.numel() * es, cur.data_ptr(),
                                        cur.numel() * es, _stream()))
    _lib.check(_lib.lib().krr_attention_quant(
        _lib.ATTN_TCGEN05, act, q.data_ptr(), nseq, KVH, G, HD, T, P, layer, 0,
        qptr.data_ptr(), vlen.data_ptr(), cptr.data_ptr(), tv.data_ptr(), out_q.data_ptr(),
        codes.data_ptr(), codes.numel(), cur.data_ptr(), cur.numel() * es, bits,
        scales.data_ptr(), _stream()))
    torch.cuda.synchronize()
    if act == _lib.BF16:
        assert torch.equal(out_q.view(torch.int16), out_ref.view(torch.int16))
    else:
        assert torch.isfinite(out_q).all()
        err = (out_q.float() - out_ref.float()).abs().max().item()
        assert err <= 4e-3 * max(1.0, out_ref.float().abs().max().item()), err
    # the expansion itself is the reference codec's dequantize_tensor (one tensor)
    from paper_2504_02921_b200 import codec
    scheme = codec.QuantScheme.INT8_PER_CHANNEL if bits == 8 else codec.QuantScheme.INT4_PER_CHANNEL
    t0 = (1 * L + layer) * 2 + 1                        # seq 1, this layer, V
    cb = codes[t0 * tb:(t0 + 1) * tb].cpu().numpy().tobytes()
    s0 = scales[t0 * KVH * HD:(t0 + 1) * KVH * HD].cpu().numpy().reshape(KVH, HD)
    ref = codec.dequantize_tensor(cb, s0, scheme, (KVH, P, HD))
    assert np.array_equal(pre[1, layer, 1].float().cpu().numpy(),
                          torch.from_numpy(ref).to(tdt).float().numpy())


def test_attention_quant_rejects_unsupported():
    """Quantised prefix pages only go through the tcgen05 kernel (head_dim 64|128)."""
    T, HD, KVH, G = 16, 256, 1, 8
    q = torch.zeros(KVH, G * T, HD, dtype=torch.float16, device="cuda")
    with pytest.raises(Exception, match="quantised prefix"):
        _lib.check(_lib.lib().krr_attention_quant(
            _lib.ATTN_TCGEN05, _lib.F16, q.data_ptr(), 1, KVH, G, HD, T, 64, 0, 0, 0, 0, 0, 0,
            q.data_ptr(), 0, 0, 0, 0, 8, 0, _stream()))
