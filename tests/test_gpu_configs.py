"""GPU parity on the BASELINE configs 2-5 at full size.

Per config and kind, on BOTH table forms (the default B-spline form and the
opt-in k-power form) and on EVERY fast kernel path (generic, per-position
TMA, line, and the window variant of the line kernel on the B-spline form --
forced with SPO_LINE / pipeline so every path runs the same full launch):

* the paths' full outputs are bitwise identical (per-position digests of
  every output bit);
* >= 2048 oracle positions per (config, kind, form, path), stratified: one
  from every 4x4x4-cell block of the grid, the first and last position of
  line-kernel runs, random ones on top (tests/strata.py), each within
  1e-5 (fp32) / 1e-12 (fp64) * sum|w*c| of the f64 oracle;
* STRICT mode bitwise equal to the reference fp32 kernels (oracle.eval_f32,
  the C restatement pinned to the reference's golden vectors) on >= 16,384
  positions of configs 2-4;
* the device-generated table equals the reference's (sha256 of the full
  reference SoA table, tests/golden/big.npz) and the golden positions'
  reference outputs;
* size-independent properties on the full workload (V == VGH.v bitwise,
  VGL gradients == VGH gradients bitwise, permutation invariance, tiled ==
  untiled, orbital shards gathered == full N).
"""
import hashlib

import numpy as np
import pytest

import oracle
from paper_1611_02665_b200.device import DeviceTable
from paper_1611_02665_b200.kernels import KernelKind, eval_form, eval_path, evaluate, streams
from paper_1611_02665_b200.multi import OrbitalPartition
from paper_1611_02665_b200.workloads import CONFIGS, config_positions
from strata import stratified_sample

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL32, TOL64 = 1e-5, 1e-12
PATHS = ("line", "window", "tma", "generic")
FORMS = ("bspline", "kpower")
N_ORACLE = 2048
N_STRICT = 16384


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available()
    return t


def as_np(out, dt, kind):
    s = streams(out, dt, kind)
    return np.stack([s[n].cpu().numpy() for n in KernelKind(kind).stream_names], axis=1)


def run_path(monkeypatch, dt, kind, pos, out, path, form):
    """evaluate() on a chosen kernel path (the same launch for every path)."""
    if path == "generic":
        evaluate(dt, kind, pos, out, pipeline=False, form=form, check=False)
        return
    monkeypatch.setenv("SPO_LINE", {"line": "1", "window": "2", "tma": "0"}[path])
    try:
        assert eval_path(dt, kind, pos.shape[0], pipeline=True, form=form) == path
        evaluate(dt, kind, pos, out, pipeline=True, form=form, check=False)
    finally:
        monkeypatch.delenv("SPO_LINE")


def digest(torch, out, P, sub=16384):
    """[P][S] int64: lane-weighted sums of the output bit patterns."""
    lanes = out.shape[2]
    w = torch.arange(1, lanes + 1, dtype=torch.int64, device=out.device)
    bits = out[:P].view(torch.int64 if out.dtype == torch.float64 else torch.int32)
    parts = [(bits[lo: lo + sub].to(torch.int64) * w).sum(-1) for lo in range(0, P, sub)]
    return torch.cat(parts)


class OracleSample:
    """f64 oracle values and scales of the sampled positions (computed once)."""

    def __init__(self, host, dt, kind, pos, sel):
        self.kind, self.sel, self.N = kind, sel, dt.n_splines
        self.ref, self.scale = oracle.eval_f64(kind, host, dt.n_splines, dt.grid.spacings, pos[sel])

    def check(self, got_rows, tol, rows=None):
        """got_rows: [len(rows)][S][N] of the sampled positions `rows` (indices into sel)."""
        rows = np.arange(len(self.sel)) if rows is None else rows
        ok, worst = oracle.tolerance_check(got_rows, self.ref[rows], self.scale[rows], tol)
        return ok, worst


def check_launches(torch, monkeypatch, dt, host, kind, pos, launch, tol, forms=FORMS, n_min=N_ORACLE):
    """All forms x paths over the full `pos` in launches of `launch`
    positions: bitwise across paths, stratified oracle sample per path."""
    P = pos.shape[0]
    sel = stratified_sample(pos, dt.grid, n_min=n_min, launch=launch)
    assert sel.size >= n_min
    osamp = OracleSample(host, dt, kind, pos, sel)
    S = KernelKind(kind).output_streams_soa
    tdt = torch.float64 if dt.dtype == np.float64 else torch.float32
    out = torch.empty((min(P, launch), S, dt.lanes), dtype=tdt, device="cuda")
    report = {}
    for form in forms:
        digests = {}
        for path in PATHS:
            if path == "window" and form == "kpower":
                continue  # the window variant reads the B-spline form only
            dg, got = [], np.empty((sel.size, S, dt.n_splines), dtype=dt.dtype)
            for lo in range(0, P, launch):
                hi = min(P, lo + launch)
                run_path(monkeypatch, dt, kind, pos[lo:hi], out, path, form)
                dg.append(digest(torch, out, hi - lo))
                mine = np.nonzero((sel >= lo) & (sel < hi))[0]
                idx = torch.from_numpy(sel[mine] - lo).cuda()
                got[mine] = as_np(out.index_select(0, idx), dt, kind)
            digests[path] = torch.cat(dg)
            ok, worst = osamp.check(got, tol)
            assert ok, (kind, form, path, worst)
            report[(form, path)] = worst
        assert torch.equal(digests["line"], digests["tma"]), (kind, form)
        if "window" in digests:
            assert torch.equal(digests["window"], digests["tma"]), (kind, form)
        assert torch.equal(digests["line"], digests["generic"]), (kind, form)
    del out
    return report


def check_strict(dt, host, kind, pos, chunk=4096):
    """STRICT mode == the reference fp32 kernels bitwise on every position."""
    for lo in range(0, pos.shape[0], chunk):
        p = pos[lo: lo + chunk]
        got = as_np(evaluate(dt, kind, p, mode="strict"), dt, kind)
        ref = oracle.eval_f32(kind, host, dt.grid.spacings, p)[:, :, : dt.n_splines]
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (kind, lo)


@pytest.mark.parametrize("tag,idx", [("cfg2", 2), ("cfg3", 3), ("cfg4", 4)])
def test_config_table_and_golden_positions(torch, golden_big, tag, idx):
    cfg = CONFIGS[idx]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)
    host = dt.reference_soa()
    assert sha(host) == str(golden_big[f"{tag}_table_sha"])
    pos = golden_big[f"{tag}_positions"]
    strict = as_np(evaluate(dt, cfg.kernel, pos, mode="strict"), dt, cfg.kernel)
    assert sha(strict) == str(golden_big[f"{tag}_f32_sha"])
    np.testing.assert_array_equal(strict[:, :, :128], golden_big[f"{tag}_f32_head"])
    fast = as_np(evaluate(dt, cfg.kernel, pos), dt, cfg.kernel)
    ref, scale = oracle.eval_f64(cfg.kernel, host, cfg.n_splines, cfg.grid.spacings, pos[:3])
    np.testing.assert_array_equal(ref[:, :, :128], golden_big[f"{tag}_f64_head"])
    np.testing.assert_array_equal(ref[:, :, -64:], golden_big[f"{tag}_f64_tail"])
    ok, worst = oracle.tolerance_check(fast[:3], ref, scale, TOL32)
    assert ok, worst


def test_config2_full_workload(torch, monkeypatch):
    cfg = CONFIGS[2]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0).with_kpower()
    host = dt.reference_soa()
    pos = config_positions(cfg)
    assert pos["vgh"].shape == (16384, 3) and pos["v"].shape == (98304, 3)
    # quadrature shells around ions near the faces leave [0,1)^3: the wrap path
    assert ((pos["v"] < 0) | (pos["v"] >= 1)).any()
    check_launches(torch, monkeypatch, dt, host, "vgh", pos["vgh"], 16384, TOL32)
    check_launches(torch, monkeypatch, dt, host, "v", pos["v"], 98304, TOL32)
    vgh = evaluate(dt, "vgh", pos["vgh"])
    assert torch.equal(evaluate(dt, "v", pos["vgh"])[:, 0], vgh[:, 0])
    check_strict(dt, host, "vgh", pos["vgh"][:N_STRICT])
    check_strict(dt, host, "v", pos["v"][:N_STRICT])


def test_config3_full_workload(torch, monkeypatch):
    cfg = CONFIGS[3]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0).with_kpower()
    host = dt.reference_soa()
    pos = config_positions(cfg)["vgl"]
    assert pos.shape == (131072, 3)
    check_launches(torch, monkeypatch, dt, host, "vgl", pos, 131072, TOL32)
    check_strict(dt, host, "vgl", pos[:N_STRICT])
    # VGL gradients are the VGH gradients bit for bit; l matches the trace
    sub = pos[:4096]
    vgl = evaluate(dt, "vgl", sub)
    vgh = evaluate(dt, "vgh", sub)
    assert torch.equal(vgl[:, :4], vgh[:, :4])
    trace = (vgh[:, 4].double() + vgh[:, 7] + vgh[:, 9])
    assert float((vgl[:, 4] - trace).abs().max() / trace.abs().max()) < 1e-5


def test_config4_full_workload(torch, monkeypatch):
    """bench.py's regime: 1,048,576 VGH positions in two 524,288-position
    launches (two per grid cell), both table forms, all three paths."""
    cfg = CONFIGS[4]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0).with_kpower()
    pos = config_positions(cfg)["vgh"]
    assert pos.shape == (1048576, 3)
    host = dt.reference_soa()
    assert eval_path(dt, "vgh", 524288) == "window" and eval_form(dt, "vgh", 524288) == "bspline"
    check_launches(torch, monkeypatch, dt, host, "vgh", pos, 524288, TOL32, n_min=4096)
    check_strict(dt, host, "vgh", pos[:N_STRICT])
    del host
    # kernel/layout invariances on one chunk
    sub = pos[:65536]
    base = evaluate(dt, "vgh", sub)
    assert bool(torch.isfinite(base.sum()))
    v = evaluate(dt, "v", sub)
    assert torch.equal(v[:, 0], base[:, 0])
    assert torch.equal(evaluate(dt, "vgl", sub)[:, :4], base[:, :4])
    perm = np.random.default_rng(7).permutation(len(sub))
    shuffled = torch.empty_like(base)
    evaluate(dt, "vgh", sub[perm], shuffled, out_index=torch.from_numpy(perm).cuda())
    assert torch.equal(shuffled, base)
    del dt
    tiled = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0, tile_size=32)
    t_out = evaluate(tiled, "vgh", sub[:8192])
    assert torch.equal(t_out, base[:8192])


def test_config5_fp64(torch, monkeypatch):
    """fp64 N=4096 normal(0,1) on 48^3, V:VGL:VGH = 12:1:1 by position index
    (2048 walkers x 128 = 262,144 positions of the mix): both forms, all
    paths, stratified oracle samples at 1e-12 * sum|w*c|."""
    cfg = CONFIGS[5]
    dt = DeviceTable.normal_f64(cfg.grid, cfg.n_splines, seed=0).with_kpower()
    host = dt.reference_soa()
    pos = config_positions(cfg, walkers=range(2048))
    for kind in ("v", "vgl", "vgh"):
        p = pos[kind]
        check_launches(torch, monkeypatch, dt, host, kind, p, p.shape[0], TOL64)


@pytest.mark.parametrize("form", FORMS)
def test_config5_orbital_shards_gather_bitwise(torch, form):
    """8 orbital shards of 512 (the config-5 partition) emulated on one GPU:
    each shard evaluates all positions; gathered == full-N bitwise."""
    cfg = CONFIGS[5]
    full = DeviceTable.normal_f64(cfg.grid, cfg.n_splines, seed=0)
    if form == "kpower":
        full.with_kpower()
    pos = config_positions(cfg, walkers=range(32))  # 4096 positions of the mix
    part = OrbitalPartition.make(cfg.n_splines, 8, quantum=16)
    for kind in ("v", "vgl", "vgh"):
        p = pos[kind]
        ref_full = evaluate(full, kind, p, form=form)[:, :, : cfg.n_splines]
        gathered = torch.empty_like(ref_full)
        for r in range(8):
            lo, hi = part.local(r)
            shard = full.slice_orbitals(lo, hi)
            if kind == "v":  # a shard generated directly (bench.py --config 5) is the same table
                direct = DeviceTable.normal_f64(cfg.grid, hi - lo, seed=0, first_spline=lo)
                assert torch.equal(direct.data, shard.data)
                del direct
            if form == "kpower":
                shard.with_kpower()
            gathered[:, :, lo:hi] = evaluate(shard, kind, p, form=form)[:, :, : hi - lo]
            del shard
        assert torch.equal(gathered, ref_full), kind
