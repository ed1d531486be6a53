"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/bspb_numba PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py [--big]

Everything stored comes from the reference's own code paths:
  * index mapping      bspb.grid._map_axis               (grid.py:109-121)
  * fp32 weights       bspb.grid._fill_axis_weights      (grid.py:124-139)
  * fp64 weights       bspb.oracle.axis_weights_f64      (oracle.py:20-42)
  * tables             bspb.coeffs.build_table + FillSpec.random (coeffs.py:80-94, 165-185)
  * positions          bspb.driver.generate_positions / _position_stream (driver.py:174-193)
  * fp32 outputs       bspb.kernels.eval_batch per position (kernels.py:445-473)
  * fp64 outputs       bspb.oracle.evaluate_f64 (oracle.py:74-115)

The fixtures are small: large arrays are pinned by sha256 instead of stored.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from bspb import coeffs, driver, grid as bgrid, kernels, oracle  # noqa: E402
from bspb.kernels import KernelKind  # noqa: E402

KINDS = (KernelKind.V, KernelKind.VGL, KernelKind.VGH)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def unit_grid(n):
    return bgrid.GridSpec(n, n, n, 1.0 / n, 1.0 / n, 1.0 / n)


def edge_xs():
    rng = np.random.default_rng(12345)
    xs = [0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, -1e-300, 1e308, -1e308,
          1e-18, -1e-18, 1.0, -1.0, 1.0 - 1e-12, 1.0 + 1e-12, 0.5, -0.25, 2.7, 47.5,
          47.999999999999, 48.0, -48.0, 1e15 + 0.3, -1e15 - 0.7, np.nextafter(1.0, 0.0),
          np.nextafter(0.0, -1.0), 123456.789, -987654.321]
    for n in (16, 48, 51, 64, 67):
        for k in range(-2, n + 3):
            x = k / n
            xs += [x, np.nextafter(x, -np.inf), np.nextafter(x, np.inf)]
    xs += list(rng.normal(0.0, 1e3, 400)) + list(rng.normal(0.0, 1e15, 200))
    xs += list(rng.random(400)) + list(rng.random(200) * 2.0 - 0.5)
    return np.array(xs, dtype=np.float64)


def make_mapping():
    xs = edge_xs()
    pairs = [(1.0 / (1.0 / n), float(n)) for n in (16, 48, 51, 64, 67)]
    pairs += [(1.0, 48.0), (1.0 / 0.25, 7.0), (1.0 / 2.0, 60.0), (1.0 / 0.5, 4.0), (1.0, 16.0)]
    i0 = np.zeros((len(pairs), xs.size), dtype=np.int64)
    t = np.zeros((len(pairs), xs.size), dtype=np.float64)
    for a, (dinv, cnt) in enumerate(pairs):
        for b, x in enumerate(xs):
            i0[a, b], t[a, b] = bgrid._map_axis(float(x), dinv, cnt)
    rng = np.random.default_rng(7)
    ts = np.concatenate([[0.0, 0.5, 0.25, 0.75, 0.125, np.nextafter(1.0, 0.0), 1e-300, 5e-324],
                         rng.random(500)])
    dinvs = np.array([1.0, 16.0, 48.0, 64.0, 2.0, 0.5, 4.0, 1.0 / 0.3])
    w32 = np.zeros((dinvs.size, ts.size, 3, 4), dtype=np.float32)
    w64 = np.zeros((dinvs.size, ts.size, 3, 4), dtype=np.float64)
    for a, dinv in enumerate(dinvs):
        for b, tt in enumerate(ts):
            bgrid._fill_axis_weights(float(tt), float(dinv), w32[a, b])
            w64[a, b] = np.array(oracle.axis_weights_f64(float(tt), 1.0 / float(dinv)))
    np.savez_compressed(os.path.join(HERE, "mapping.npz"), xs=xs,
                        pairs=np.array(pairs), i0=i0, t=t, ts=ts, dinvs=dinvs, w32=w32, w64=w64)
    print("mapping.npz", xs.size, "x values,", len(pairs), "grids")


def ref_f32(table, kind, pos):
    """[P][S][N] float32 through the reference production kernels, one call per position."""
    out = kernels.allocate_outputs(table)
    rows = []
    for p in pos:
        kernels.eval_batch(table, kind, p, out)
        st = kernels.collect_streams(out, kind)
        rows.append(np.stack([st[name] for name in kind.stream_names]))
    return np.stack(rows).astype(np.float32)


def ref_f64(table, kind, pos):
    rows = []
    for p in pos:
        st = oracle.evaluate_f64(table, kind, p)
        rows.append(np.stack([st[name] for name in kind.stream_names]))
    return np.stack(rows)


def make_cfg1():
    g = unit_grid(16)
    table = coeffs.build_table(g, 64, coeffs.FillSpec.random(0))
    pos = driver.generate_positions(1, 0, 0, 512, g).vgh
    edge = np.array([[1 - 1e-6] * 3, [-0.01, 1.02, 0.5], [0.0, 0.0, 0.0],
                     [1.0, 1.0, 1.0], [-1e-18, 0.999999999999, 17.25]])
    d = dict(table_sha=sha(table.data), table_shape=np.array(table.data.shape),
             positions=pos, edge_positions=edge)
    for kind in KINDS:
        f32 = ref_f32(table, kind, pos)
        d[f"{kind.value}_f32_sha"] = sha(f32)
        d[f"{kind.value}_f32_head"] = f32[:64]
        d[f"{kind.value}_f32_edge"] = ref_f32(table, kind, edge)
        d[f"{kind.value}_f64_head"] = ref_f64(table, kind, pos[:24])
        d[f"{kind.value}_f64_edge"] = ref_f64(table, kind, edge)
    # a tiled variant (tile_size 16 -> M=4) must give the same bits (test_kernels.py:62-75)
    tiled = coeffs.tile_table(table, 16)
    d["vgh_f32_tiled_sha"] = sha(ref_f32(tiled, KernelKind.VGH, pos))
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **d)
    print("cfg1.npz", {k: (v.shape if hasattr(v, "shape") else v) for k, v in d.items()})


def small_cases():
    """Ragged / tiny tables (N=5, 24, 33) on non-cubic grids, fp32 + f64."""
    out = {}
    for tag, (counts, spac, n, seed) in {
        "ragged5": ((12, 12, 12), (1.0, 1.0, 1.0), 5, 4),
        "g12n24": ((12, 12, 12), (1.0, 1.0, 1.0), 24, 42),
        "g5x4x6n7": ((5, 4, 6), (1.0, 1.0, 1.0), 7, 3),
        "g8n33": ((8, 9, 10), (0.5, 0.25, 2.0), 33, 9),
    }.items():
        g = bgrid.GridSpec(*counts, *spac)
        table = coeffs.build_table(g, n, coeffs.FillSpec.random(seed))
        rng = np.random.default_rng(seed)
        pos = rng.random((16, 3)) * np.asarray(g.lengths) * 3.0 - np.asarray(g.lengths)
        out[f"{tag}_positions"] = pos
        out[f"{tag}_meta"] = np.array([*counts, n, seed], dtype=np.int64)
        out[f"{tag}_spacing"] = np.array(spac)
        out[f"{tag}_table_sha"] = sha(table.data)
        for kind in KINDS:
            out[f"{tag}_{kind.value}_f32"] = ref_f32(table, kind, pos)
            out[f"{tag}_{kind.value}_f64"] = ref_f64(table, kind, pos)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small.npz", len(out), "arrays")


def make_big():
    """Full-size tables of configs 2-4: table hashes + a few sampled positions."""
    out = {}
    for tag, n_grid, n_spl, kind, walkers in (
        ("cfg2", 48, 512, KernelKind.VGH, 256),
        ("cfg3", 48, 2048, KernelKind.VGL, 1024),
        ("cfg4", 64, 4096, KernelKind.VGH, 4096),
    ):
        t0 = time.time()
        g = unit_grid(n_grid)
        table = coeffs.build_table(g, n_spl, coeffs.FillSpec.random(0))
        out[f"{tag}_table_sha"] = sha(table.data)
        # walker 0 and the last walker, the first 4 moves of iteration 0
        pos = np.concatenate([
            driver._position_stream(1, 0, 0, driver._KERNEL_STREAM_ID[kind], 4, g),
            driver._position_stream(1, walkers - 1, 0, driver._KERNEL_STREAM_ID[kind], 4, g),
        ])
        out[f"{tag}_positions"] = pos
        f32 = ref_f32(table, kind, pos)
        out[f"{tag}_f32_sha"] = sha(f32)
        out[f"{tag}_f32_head"] = f32[:, :, :128]
        f64 = ref_f64(table, kind, pos[:3])
        out[f"{tag}_f64_head"] = f64[:, :, :128]
        out[f"{tag}_f64_sum"] = f64.sum(axis=2)
        # a 4th-corner sample so tests can spot-check the whole orbital range
        out[f"{tag}_f64_tail"] = f64[:, :, -64:]
        print(tag, "built+evaluated in %.1fs" % (time.time() - t0), flush=True)
        del table
    np.savez_compressed(os.path.join(HERE, "big.npz"), **out)


def make_philox_pins():
    """numpy Philox streams as the reference consumes them (coeffs.py:91-94,
    driver.py:174-179); pins the product's on-device generators."""
    g = unit_grid(16)
    d = {}
    for n in (0, 1, 63, 4095):
        d[f"fill_s0_n{n}"] = coeffs.FillSpec.random(0).spline_values(g, n)
    d["fill_s7_n5_g5x4x6"] = coeffs.FillSpec.random(7).spline_values(bgrid.GridSpec(5, 4, 6), 5)
    d["pos_s1_w3_i2_k2"] = driver._position_stream(1, 3, 2, 2, 37, g)
    d["pos_s1_w4095_i0_k2"] = driver._position_stream(1, 4095, 0, 2, 256, unit_grid(64))
    np.savez_compressed(os.path.join(HERE, "philox.npz"), **d)
    print("philox.npz", list(d))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also build configs 2-4 (minutes)")
    args = ap.parse_args()
    make_mapping()
    make_cfg1()
    small_cases()
    make_philox_pins()
    if args.big:
        make_big()
