"""ORACLE / TEST INFRASTRUCTURE ONLY -- generates tests/golden/ fixtures by
running the unmodified reference (oracle/_ref, built from /root/reference) on
the seeded BASELINE inputs.  Run here (where /root/reference exists):

    python oracle/make_golden.py small      # seconds: CPU-test fixtures
    python oracle/make_golden.py c1 c2      # full BASELINE C1 / C2 solves (C2 ~ 10 min)
    python oracle/make_golden.py capped200:c3   # BASELINE-size capped-parity solve (lsqr_cap = 200)
    python oracle/make_golden.py cappedulp200:c3  # same, b moved one ulp (the reference's own sensitivity)
    python oracle/make_golden.py curg:c3    # full-size Gaussian-shim CurState steps (first augments)

Capped and Gaussian fixtures generate their inputs with the oracle's own
generator (ref.Problem.generate, byte-identical to the product's), so no copy
of a 20 GB matrix is made.

The fixtures are small .npz files (indices, rho history, phase iterations,
x, residuals, trace heads) so tests on the GPU box never need /root/reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_05065_b200 as apc  # noqa: E402  (host-side generator only)
from oracle import ref  # noqa: E402

GOLD = Path(os.environ.get("APC_GOLD_DIR", ROOT / "tests" / "golden"))

# the solver settings each config is run with
BASELINE_SOLVER = {
    1: dict(mu=0.0, block=20, eps_lsqr=1e-8, seed=1),
    2: dict(mu=1e-6, block=50, eps_lsqr=1e-8, max_rank=200, seed=1),
    3: dict(mu=1e-4, block=100, eps_lsqr=1e-8, eps_cur=3e-3, max_rank=1000, seed=1),
    4: dict(mu=0.0, block=250, eps_lsqr=1e-10, max_rank=250, seed=1),
    5: dict(mu=1e-8, block=250, eps_lsqr=1e-8, eps_cur=3e-7, max_rank=500, seed=1),
}


def _save(name: str, **arrays):
    GOLD.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(GOLD / f"{name}.npz", **arrays)
    print("wrote", GOLD / f"{name}.npz", flush=True)


def solve_fixture(name, cfgid, m, n, knobs, plain=False):
    p = apc.Problem(cfgid, m, n)
    rp = ref.Problem.from_apc(p)
    t0 = time.time()
    r = ref.solve(rp, p.b, dict(knobs, trace_sample_stride=0), plain=plain)
    wall = time.time() - t0
    _save(name, x=r.x, status=r.status, final_rho=r.final_rho, final_relres=r.final_relres,
          system_matvecs=r.system_matvecs, row_indices=r.row_indices, col_indices=r.col_indices,
          rho_history=r.rho_history, phase_rank=r.phase_rank, phase_iters=r.phase_iters,
          phase_reason=r.phase_reason, phase_rho=r.phase_rho, phase_relres=r.phase_relres,
          phase_t_lsqr_ms=r.phase_t_lsqr_ms, phase_t_total_ms=r.phase_t_total_ms,
          trace_phibar_head=r.trace_phibar[:64], wall_s=wall,
          meta=json.dumps(dict(config=cfgid, m=m, n=n, knobs=knobs, plain=plain)))
    return r, wall


def small():
    # reference known answers used by the CPU suite (port pinning) and GPU tests
    rng = np.random.default_rng(20260415)
    # RNG streams
    _save("rng", u64=ref.rng(20260416, 0, 256, stream=3, index=9), gauss=ref.rng(20260416, 2, 256, stream=2),
          below=ref.rng(7, 3, 256, bound=1000003), mix=np.array([ref.mix64(x) for x in (0, 1, 12345)], np.uint64))
    # sparse-sign embedding and sketches
    rows, signs, scale = ref.sparse_sign(11, 300, 8, ref.mix64(1 ^ 0x5CE7C3A1B2D4F688))
    A = rng.standard_normal((300, 40))
    A[rng.random(A.shape) < 0.5] = 0.0
    Y = ref.sketch_sparse_sign(ref.Problem.from_numpy(A), 11, 8, ref.mix64(1 ^ 0x5CE7C3A1B2D4F688))
    Ys = ref.sketch_sparse_sign(ref.Problem.from_numpy(A, sparse=True), 11, 8, 99)
    Ya = ref.sketch_sparse_sign(ref.Problem.from_numpy(A), 11, 8, 5, mu=0.25, augmented=True)
    _save("sketch", rows=rows, signs=signs, scale=scale, A=A, Y=Y, Ys=Ys, Ya=Ya)
    # LUPP known answers (ties, zero columns, random)
    cases = {}
    for k, W in enumerate([rng.standard_normal((50, 12)), np.ones((6, 4)), np.zeros((5, 3)),
                           np.where(rng.random((40, 9)) < 0.4, 0.0, rng.standard_normal((40, 9)))]):
        o, mg = ref.lupp(W, -1)
        cases[f"W{k}"], cases[f"o{k}"], cases[f"m{k}"] = W, o, mg
    _save("lupp", **cases)
    # matvec known answers (dense, CSC, augmented)
    x = rng.standard_normal(40)
    u = rng.standard_normal(340)
    rp, rs = ref.Problem.from_numpy(A), ref.Problem.from_numpy(A, sparse=True)
    _save("matvec", A=A, x=x, u=u, y=ref.matvec(rp, x), ys=ref.matvec(rs, x), g=ref.matvec(rp, u[:300], transpose=True),
          gs=ref.matvec(rs, u[:300], transpose=True), ya=ref.matvec(rp, x, 0.3, True),
          ga=ref.matvec(rs, u, 0.3, True, True))
    # LSQR and full solves on small BASELINE-shaped inputs
    solve_fixture("plain_c2_small", 2, 3000, 300, dict(mu=1e-3, eps_lsqr=1e-10, lsqr_cap=300), plain=True)
    solve_fixture("solve_c1_small", 1, 400, 50, dict(mu=0.0, eps_lsqr=1e-8, block=5, seed=1))
    solve_fixture("solve_c2_small", 2, 4000, 400, dict(mu=1e-3, eps_lsqr=1e-10, block=8, seed=3, max_rank=40))
    cur = ref.cur_steps(ref.Problem.from_apc(apc.Problem(2, 3000, 300)), 7, 7, 6)
    _save("cur_c2_small", I=cur["I"], J=cur["J"], rho=cur["rho"], added=cur["added"])


def capped_fixture(k: int, cap: int, ulp: bool = False):
    """SURVEY.md 8(c)(3) capped-parity mode at BASELINE size: the reference
    aplicur_solve (solver.hpp:162-392) with the BASELINE knobs plus lsqr_cap."""
    knobs = dict(BASELINE_SOLVER[k], trace_sample_stride=0, lsqr_cap=cap)
    t0 = time.time()
    p = ref.Problem.generate(k)
    gen_s = time.time() - t0
    b = np.nextafter(p.b, np.inf) if ulp else None
    t0 = time.time()
    r = ref.solve(p, b, knobs, consume=True)
    wall = time.time() - t0
    p.free()
    lsqr_s = float(np.sum(r.phase_t_lsqr_ms)) / 1e3
    common = dict(phase_rank=r.phase_rank, phase_iters=r.phase_iters, phase_reason=r.phase_reason,
                  trace_phibar=r.trace_phibar, final_relres=r.final_relres, status=r.status,
                  row_indices=r.row_indices, col_indices=r.col_indices, wall_s=wall, gen_s=gen_s,
                  lsqr_s=lsqr_s, setup_s=wall - lsqr_s,
                  meta=json.dumps(dict(config=k, cap=cap, knobs=knobs, ulp=ulp, threads=1)))
    if ulp and os.environ.get("APC_ULP_RAW"):  # concurrent run: keep x, the pair step measures the sensitivity
        _save(f"capped_c{k}_k{cap}_ulpraw", x=r.x, **common)
    elif ulp:  # x itself is only needed to measure the sensitivity against the main fixture
        main = np.load(GOLD / f"capped_c{k}_k{cap}.npz")
        xs = float(np.linalg.norm(r.x - main["x"]) / np.linalg.norm(main["x"]))
        ph = r.trace_phibar
        mp = main["trace_phibar"]
        nn = min(len(ph), len(mp))
        _save(f"capped_c{k}_k{cap}_ulp", x_sens=xs,
              phibar_sens=float(np.max(np.abs(ph[:nn] - mp[:nn]) / np.abs(mp[:nn]))), **common)
    else:
        _save(f"capped_c{k}_k{cap}", x=r.x, final_rho=r.final_rho, system_matvecs=r.system_matvecs,
              rho_history=r.rho_history, phase_rho=r.phase_rho, phase_sigma_hat=r.phase_sigma_hat,
              phase_relres=r.phase_relres, phase_t_lsqr_ms=r.phase_t_lsqr_ms,
              phase_t_total_ms=r.phase_t_total_ms, trace_phase=r.trace_phase, trace_iter=r.trace_iter,
              trace_matvecs=r.trace_matvecs, **common)
    print(f"capped C{k} cap {cap} ulp {ulp}: wall {wall:.1f}s (gen {gen_s:.1f}s) ranks {r.phase_rank} "
          f"iters {r.phase_iters} reasons {r.phase_reason} relres {r.final_relres}", flush=True)


def capped_ensemble_member(k: int, cap: int, seed: int, ulps: int = 1):
    """The reference's own run-to-run spread of the stop-rule iteration counts:
    the capped solve (same knobs, lsqr_cap = cap) on b with EVERY entry moved
    one ulp up or down (signs from `seed`) -- a rounding-level perturbation like
    a different summation order.  Only the phase iteration counts and stop
    reasons before the cap are used (tests/test_gpu_baseline_capped.py)."""
    knobs = dict(BASELINE_SOLVER[k], trace_sample_stride=0, lsqr_cap=cap)
    p = ref.Problem.generate(k)
    sgn = np.random.default_rng(seed).integers(0, 2, size=p.b.shape[0]) * 2 - 1
    b = p.b + sgn * ulps * np.spacing(p.b) if ulps > 1 else np.where(
        sgn > 0, np.nextafter(p.b, np.inf), np.nextafter(p.b, -np.inf))
    t0 = time.time()
    r = ref.solve(p, b, knobs, consume=True)
    wall = time.time() - t0
    p.free()
    _save(f"capped_c{k}_ens{seed}" + (f"u{ulps}" if ulps > 1 else ""), phase_rank=r.phase_rank, phase_iters=r.phase_iters,
          phase_reason=r.phase_reason, trace_phibar=r.trace_phibar, wall_s=wall,
          meta=json.dumps(dict(config=k, cap=cap, knobs=knobs, seed=seed, ulps=ulps,
                               perturbation=f"every b_i moved {ulps} ulp up or down")))
    print(f"ensemble C{k} seed {seed} ulps {ulps}: wall {wall:.1f}s iters {r.phase_iters} reasons {r.phase_reason}", flush=True)


def capped_ensemble_collect(k: int):
    """Merge the members into capped_c{k}_ens.npz (rows = members)."""
    fs = sorted(GOLD.glob(f"capped_c{k}_ens[0-9]*.npz"))
    if not fs:
        raise RuntimeError(f"no ensemble members for C{k}")
    ms = [np.load(f) for f in fs]
    nph = min(len(m["phase_iters"]) for m in ms)
    _save(f"capped_c{k}_ens", phase_iters=np.array([m["phase_iters"][:nph] for m in ms]),
          phase_reason=np.array([m["phase_reason"][:nph] for m in ms]),
          phase_rank=np.array([m["phase_rank"][:nph] for m in ms]),
          seeds=np.array([json.loads(str(m["meta"]))["seed"] for m in ms]),
          ulps=np.array([json.loads(str(m["meta"])).get("ulps", 1) for m in ms]), meta=str(ms[0]["meta"]))
    for f in fs:
        f.unlink()


def capped_pair(k: int, cap: int):
    """Main and one-ulp capped runs side by side (host RAM permitting: C5's
    reference solve peaks near 65 GB), then the sensitivity fixture."""
    env = dict(os.environ, APC_ULP_RAW="1")
    me = Path(__file__).resolve()
    pm = subprocess.Popen([sys.executable, str(me), f"capped{cap}:c{k}"])
    pu = subprocess.Popen([sys.executable, str(me), f"cappedulp{cap}:c{k}"], env=env)
    if pm.wait() != 0 or pu.wait() != 0:
        raise RuntimeError("capped pair failed")
    main = np.load(GOLD / f"capped_c{k}_k{cap}.npz")
    raw = dict(np.load(GOLD / f"capped_c{k}_k{cap}_ulpraw.npz"))
    x = raw.pop("x")
    ph, mp = raw["trace_phibar"], main["trace_phibar"]
    nn = min(len(ph), len(mp))
    _save(f"capped_c{k}_k{cap}_ulp", x_sens=float(np.linalg.norm(x - main["x"]) / np.linalg.norm(main["x"])),
          phibar_sens=float(np.max(np.abs(ph[:nn] - mp[:nn]) / np.abs(mp[:nn]))), **raw)
    (GOLD / f"capped_c{k}_k{cap}_ulpraw.npz").unlink()


def gaussian_cur_fixture(k: int, steps: int = 3):
    """Full-size CurState init/augment/refresh steps (cur.hpp:209-315) with the
    Gaussian shim sketch (sketch.hpp:173-197), the BASELINE block of config k."""
    block = BASELINE_SOLVER[k]["block"]
    t0 = time.time()
    p = ref.Problem.generate(k)
    gen_s = time.time() - t0
    t0 = time.time()
    cur = ref.cur_steps(p, block, 1, steps, gaussian=True)
    wall = time.time() - t0
    Y = np.ascontiguousarray(cur["Y"].T)  # column-major bytes of Y (s x n)
    E = np.ascontiguousarray(cur["eres"].T)
    extra = dict(Y=cur["Y"]) if cur["Y"].size <= 200000 else {}
    _save(f"curg_c{k}", I=cur["I"], J=cur["J"], rho=cur["rho"], added=cur["added"],
          y_sha256=hashlib.sha256(Y.tobytes()).hexdigest(), eres_sha256=hashlib.sha256(E.tobytes()).hexdigest(),
          y_col0=cur["Y"][:, 0].copy(), y_fro=float(np.linalg.norm(cur["Y"])), wall_s=wall, gen_s=gen_s,
          meta=json.dumps(dict(config=k, block=block, steps=steps, seed=1, gaussian=True)), **extra)
    p.free()
    print(f"curg C{k}: {wall:.1f}s rank {len(cur['I'])} rho {cur['rho']}", flush=True)


def main(argv):
    if not ref.available():
        ref.build()
    for what in argv or ["small"]:
        if what == "small":
            small()
        elif what.startswith("ens") and what.count(":") in (2, 3):  # ens<cap>:c<k>:<seed>[:<ulps>]
            head, c, s, *u = what.split(":")
            capped_ensemble_member(int(c[1:]), int(head[3:]), int(s), int(u[0]) if u else 1)
        elif what.startswith("enscollect:c"):
            capped_ensemble_collect(int(what[len("enscollect:c"):]))
        elif what.startswith("cappedpair") and ":c" in what:
            head, c = what.split(":c")
            capped_pair(int(c), int(head[len("cappedpair"):] or 200))
        elif what.startswith("capped") and ":c" in what:
            head, c = what.split(":c")
            ulp = head.startswith("cappedulp")
            capped_fixture(int(c), int(head[len("cappedulp" if ulp else "capped"):] or 200), ulp=ulp)
        elif what.startswith("curg:c"):
            gaussian_cur_fixture(int(what[6:]))
        elif what.startswith("sens"):
            # the reference's own x sensitivity: rerun with b moved by one ulp
            k = int(what[4:])
            p = apc.Problem(k)
            t0 = time.time()
            r = ref.solve(ref.Problem.from_apc(p), np.nextafter(p.b, np.inf),
                          dict(BASELINE_SOLVER[k], trace_sample_stride=0))
            _save(f"baseline_c{k}_ulp", x=r.x, row_indices=r.row_indices, phase_iters=r.phase_iters,
                  final_relres=r.final_relres, wall_s=time.time() - t0)
        elif what.startswith("c") and what[1:].isdigit():
            k = int(what[1:])
            r, wall = solve_fixture(f"baseline_c{k}", k, 0, 0, BASELINE_SOLVER[k])
            print(f"C{k}: wall {wall:.1f}s status {r.status} rank {len(r.row_indices)} iters {r.phase_iters} "
                  f"relres {r.final_relres}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
