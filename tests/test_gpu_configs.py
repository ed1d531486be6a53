"""GPU parity on the BASELINE configs 2-5 at full size.

Per config: the device-generated table equals the reference's table (sha256
of the reference SoA layout, from tests/golden/big.npz); strict mode equals
the reference fp32 kernels bitwise on the golden positions; fast mode is
within 1e-5 * sum|w*c| (fp32) / 1e-12 (fp64) of the f64 oracle on seeded
samples of the full workload; size-independent properties hold on the full
workload (V == VGH.v bitwise, VGL gradients == VGH gradients bitwise,
pipelined == generic, tiled == untiled, permutation invariance,
orbital-sharded == full-N)."""
import hashlib

import numpy as np
import pytest

import oracle
from paper_1611_02665_b200.device import DeviceTable
from paper_1611_02665_b200.kernels import KernelKind, evaluate, streams
from paper_1611_02665_b200.multi import OrbitalPartition
from paper_1611_02665_b200.workloads import CONFIGS, config_positions

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL32, TOL64 = 1e-5, 1e-12


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


def check_sample(dt, host, kind, pos, tol, mode="fast"):
    got = as_np(evaluate(dt, kind, pos, mode=mode), dt, kind)
    ref, scale = oracle.eval_f64(kind, host, dt.n_splines, dt.grid.spacings, pos)
    ok, worst = oracle.tolerance_check(got, ref, scale, tol)
    assert ok, (kind, worst)
    return worst


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


def test_config2_full_workload(torch):
    cfg = CONFIGS[2]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)
    host = dt.reference_soa()
    pos = config_positions(cfg)
    assert pos["vgh"].shape == (16384, 3) and pos["v"].shape == (98304, 3)
    vgh = evaluate(dt, "vgh", pos["vgh"])
    v = evaluate(dt, "v", pos["vgh"])
    assert torch.equal(v[:, 0], vgh[:, 0])
    vq = evaluate(dt, "v", pos["v"])
    assert torch.isfinite(vq).all() and torch.isfinite(vgh).all()
    rng = np.random.default_rng(21)
    check_sample(dt, host, "vgh", pos["vgh"][rng.choice(16384, 48, replace=False)], TOL32)
    qs = pos["v"][rng.choice(98304, 64, replace=False)]
    check_sample(dt, host, "v", qs, TOL32)
    # quadrature shells around ions near the faces leave [0,1)^3: the wrap path
    assert ((pos["v"] < 0) | (pos["v"] >= 1)).any()
    sel = rng.choice(98304, 64, replace=False)
    ref, scale = oracle.eval_f64("v", host, 512, cfg.grid.spacings, pos["v"][sel])
    ok, worst = oracle.tolerance_check(vq[sel][:, :, :512].cpu().numpy(), ref, scale, TOL32)
    assert ok, worst


def test_config3_full_workload(torch):
    cfg = CONFIGS[3]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)
    pos = config_positions(cfg)["vgl"]
    assert pos.shape == (131072, 3)
    out = torch.empty((65536, 5, dt.lanes), dtype=torch.float32, device="cuda")
    host = dt.reference_soa()
    rng = np.random.default_rng(3)
    for lo in (0, 65536):
        chunk = pos[lo: lo + 65536]
        evaluate(dt, "vgl", chunk, out)
        sel = rng.choice(65536, 16, replace=False)
        ref, scale = oracle.eval_f64("vgl", host, 2048, cfg.grid.spacings, chunk[sel])
        ok, worst = oracle.tolerance_check(out[sel].cpu().numpy(), ref, scale, TOL32)
        assert ok, worst
    # VGL gradients are the VGH gradients bit for bit; l matches the trace
    sub = pos[:4096]
    vgl = evaluate(dt, "vgl", sub)
    vgh = evaluate(dt, "vgh", sub)
    assert torch.equal(vgl[:, :4], vgh[:, :4])
    trace = (vgh[:, 4].double() + vgh[:, 7] + vgh[:, 9])
    assert float((vgl[:, 4] - trace).abs().max() / trace.abs().max()) < 1e-5


def test_config4_full_workload(torch):
    cfg = CONFIGS[4]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0)
    pos = config_positions(cfg)["vgh"]
    assert pos.shape == (1048576, 3)
    chunk = 65536
    out = torch.empty((chunk, 10, dt.lanes), dtype=torch.float32, device="cuda")
    host = dt.reference_soa()
    rng = np.random.default_rng(4)
    checksum = 0.0
    for lo in range(0, len(pos), chunk):
        evaluate(dt, "vgh", pos[lo: lo + chunk], out)
        assert bool(torch.isfinite(out).all())
        checksum += float(out[:, 0].double().sum())
        if lo // chunk in (0, 7, 15):
            sel = rng.choice(chunk, 8, replace=False)
            ref, scale = oracle.eval_f64("vgh", host, 4096, cfg.grid.spacings, pos[lo + sel])
            ok, worst = oracle.tolerance_check(out[sel].cpu().numpy(), ref, scale, TOL32)
            assert ok, worst
    assert np.isfinite(checksum)
    # kernel/layout invariances on one chunk
    sub = pos[:chunk]
    base = evaluate(dt, "vgh", sub)
    assert torch.equal(base, evaluate(dt, "vgh", sub, pipeline=False))
    v = evaluate(dt, "v", sub)
    assert torch.equal(v[:, 0], base[:, 0])
    perm = np.random.default_rng(7).permutation(chunk)
    shuffled = torch.empty_like(base)
    evaluate(dt, "vgh", sub[perm], shuffled, out_index=torch.from_numpy(perm).cuda())
    assert torch.equal(shuffled, base)
    del host
    tiled = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0, tile_size=32)
    t_out = evaluate(tiled, "vgh", sub[:8192])
    assert torch.equal(t_out, base[:8192])


def test_config5_fp64_orbital_sharded(torch):
    """fp64 N=4096 normal(0,1) on 48^3, 8 orbital shards of 512 emulated on
    one GPU: each shard evaluates all positions; the gathered shards equal
    the full-N evaluation bit for bit and sit within 1e-12 * sum|w*c| of the
    f64 oracle.  V:VGL:VGH = 12:1:1 by position index."""
    cfg = CONFIGS[5]
    full = DeviceTable.normal_f64(cfg.grid, cfg.n_splines, seed=0)
    pos = config_positions(cfg, walkers=range(32))  # 4096 positions of the mix
    part = OrbitalPartition.make(cfg.n_splines, 8, quantum=16)
    host = full.reference_soa()
    for kind in ("v", "vgl", "vgh"):
        p = pos[kind]
        ref_full = evaluate(full, kind, p)[:, :, : cfg.n_splines]
        gathered = torch.empty_like(ref_full)
        for r in range(8):
            lo, hi = part.local(r)
            shard = full.slice_orbitals(lo, hi)
            gathered[:, :, lo:hi] = evaluate(shard, kind, p)[:, :, : hi - lo]
            del shard
        assert torch.equal(gathered, ref_full)
        sel = np.random.default_rng(5).choice(len(p), 8, replace=False)
        ref, scale = oracle.eval_f64(kind, host, cfg.n_splines, cfg.grid.spacings, p[sel])
        ok, worst = oracle.tolerance_check(ref_full[sel].cpu().numpy(), ref, scale, TOL64)
        assert ok, (kind, worst)


def test_config4_full_workload_kpower(torch):
    """bench.py's exact regime: config 4 on the k-power table form in
    524,288-position launches (line kernel): every output finite, sampled
    positions of every launch within 1e-5 * sum|w*c| of the f64 oracle, and
    the size-independent identities on the k-power form (V == VGH.v, VGL
    gradients == VGH gradients, pipelined == generic, permutation
    invariance) bitwise."""
    from paper_1611_02665_b200.kernels import eval_form, eval_path

    cfg = CONFIGS[4]
    dt = DeviceTable.random(cfg.grid, cfg.n_splines, seed=0).with_kpower()
    pos = config_positions(cfg)["vgh"]
    chunk = 524288
    assert eval_path(dt, "vgh", chunk) == "line" and eval_form(dt, "vgh", chunk) == "kpower"
    out = torch.empty((chunk, 10, dt.lanes), dtype=torch.float32, device="cuda")
    host = dt.reference_soa()
    rng = np.random.default_rng(44)
    for lo in range(0, len(pos), chunk):
        evaluate(dt, "vgh", pos[lo: lo + chunk], out)
        assert bool(torch.isfinite(out.sum()))  # any NaN/inf poisons the (fp32, no temporary) sum
        sel = rng.choice(chunk, 12, replace=False)
        ref, scale = oracle.eval_f64("vgh", host, 4096, cfg.grid.spacings, pos[lo + sel])
        ok, worst = oracle.tolerance_check(out[sel].cpu().numpy(), ref, scale, TOL32)
        assert ok, worst
    del out, host
    sub = pos[:65536]
    base = evaluate(dt, "vgh", sub, form="kpower")
    assert torch.equal(base, evaluate(dt, "vgh", sub, form="kpower", pipeline=False))
    assert torch.equal(evaluate(dt, "v", sub, form="kpower")[:, 0], base[:, 0])
    assert torch.equal(evaluate(dt, "vgl", sub, form="kpower")[:, 1:4], base[:, 1:4])
    perm = np.random.default_rng(9).permutation(len(sub))
    shuffled = torch.empty_like(base)
    evaluate(dt, "vgh", sub[perm], shuffled, out_index=torch.from_numpy(perm).cuda(), form="kpower")
    assert torch.equal(shuffled, base)


def test_config5_fp64_orbital_sharded_kpower(torch):
    """Config 5 on the k-power form: 8 orbital shards (each its own k-power
    table) gathered == the full-N k-power evaluation bitwise, within 1e-12 *
    sum|w*c| of the f64 oracle."""
    cfg = CONFIGS[5]
    full = DeviceTable.normal_f64(cfg.grid, cfg.n_splines, seed=0).with_kpower()
    pos = config_positions(cfg, walkers=range(32))
    part = OrbitalPartition.make(cfg.n_splines, 8, quantum=16)
    host = full.reference_soa()
    for kind in ("v", "vgl", "vgh"):
        p = pos[kind]
        ref_full = evaluate(full, kind, p, form="kpower")[:, :, : cfg.n_splines]
        gathered = torch.empty_like(ref_full)
        for r in range(8):
            lo, hi = part.local(r)
            shard = full.slice_orbitals(lo, hi).with_kpower()
            gathered[:, :, lo:hi] = evaluate(shard, kind, p, form="kpower")[:, :, : hi - lo]
            del shard
        assert torch.equal(gathered, ref_full)
        sel = np.random.default_rng(6).choice(len(p), 8, replace=False)
        ref, scale = oracle.eval_f64(kind, host, cfg.n_splines, cfg.grid.spacings, p[sel])
        ok, worst = oracle.tolerance_check(ref_full[sel].cpu().numpy(), ref, scale, TOL64)
        assert ok, (kind, worst)
