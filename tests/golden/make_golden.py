"""Generate golden vectors by running the REFERENCE package (abft_guard 0.1.0).

Run in the build container only (the reference is not present on GPU boxes):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz / *.json

The fixtures pin both the oracle (oracle/abft_oracle.py) and the B200 path:
inputs are seeded, outputs/verdicts come from the reference's own
``execute`` / ``run_protected_pipeline`` / ``global_abft_check`` / ``select``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import abft_guard  # noqa: F401
    from abft_guard import checksum, cost, shapes, tiled
    return checksum, cost, shapes, tiled


def _tiling_dict(t):
    return dict(tb_m=t.tb_m, tb_n=t.tb_n, warp_m=t.warp_m, warp_n=t.warp_n,
                thread_m=t.thread_m, thread_n=t.thread_n, k_step=t.k_step)


def make_execute_cases(tiled, shapes):
    T = tiled.TilingConfig
    tilings = {
        "default": T(),
        "small": T(tb_m=16, tb_n=16, warp_m=8, warp_n=8, thread_m=8, thread_n=8, k_step=2),
        "t64": T(tb_m=64, tb_n=64, warp_m=32, warp_n=32, thread_m=16, thread_n=8, k_step=2),
        "t4x4": T(tb_m=32, tb_n=32, warp_m=16, warp_n=16, thread_m=4, thread_n=4, k_step=2),
        "t2x2k1": T(tb_m=32, tb_n=16, warp_m=16, warp_n=16, thread_m=2, thread_n=2, k_step=1),
        "t6x6k3": T(tb_m=48, tb_n=48, warp_m=24, warp_n=24, thread_m=6, thread_n=6, k_step=3),
        "t16x16": T(tb_m=128, tb_n=128, warp_m=64, warp_n=64, thread_m=16, thread_n=16, k_step=2),
    }
    rng = np.random.default_rng(20261017)
    cases = []
    inputs = {}    # id(a) -> input-set key (a, b stored once per set)
    outputs = {}   # (input key, fault key) -> output stored once (scheme-independent)

    def add(name, a, b, tiling_name, scheme, faults, dtype):
        rep = tiled.execute(a, b, tilings[tiling_name], scheme, faults=faults, dtype=dtype)
        fl = []
        for f in faults:
            if isinstance(f, tiled.OutputFault):
                fl.append(["output", f.row, f.col, float(f.delta)])
            else:
                fl.append(["thread-mma", f.thread_row, f.thread_col, f.step, f.local_index, float(f.delta)])
        meta = dict(name=name, tiling=tiling_name, tiling_fields=_tiling_dict(tilings[tiling_name]),
                    scheme=scheme.value, faults=fl, dtype=dtype.tag.value if dtype else None,
                    detected=bool(rep.detected),
                    op_counts=[rep.op_counts.base_mma_count, rep.op_counts.redundant_mma_count,
                               rep.op_counts.checksum_op_count],
                    padded=[rep.padded_shape.m, rep.padded_shape.n, rep.padded_shape.k])
        if scheme is tiled.Scheme.GLOBAL_ABFT:
            v = rep.verdicts[0]
            meta["global"] = [bool(v.detected), float(v.lhs), float(v.rhs), float(v.tolerance_used)]
            tv = np.zeros((0, 5))
        else:
            tv = np.array([[v.thread_row, v.thread_col, float(v.detected), v.max_abs_diff, v.tolerance_used]
                           for v in rep.verdicts], dtype=np.float64).reshape(-1, 5)
        arrays = dict(tv=tv)
        key = inputs.get(id(a))
        if key is None:
            key = inputs[id(a)] = f"in{len(inputs)}"
            arrays["a"], arrays["b"] = a, b
        meta["inputs"] = key
        okey = (key, json.dumps(fl), tiling_name)
        if okey not in outputs:
            outputs[okey] = f"out{len(outputs)}"
            arrays["out"] = np.asarray(rep.output)
        meta["output"] = outputs[okey]
        cases.append((meta, arrays))

    S = tiled.Scheme
    all_schemes = list(S)
    # exact-int cases (bit-exact parity)
    for (m, n, k), tl in [((16, 16, 16), "default"), ((23, 17, 9), "small"), ((64, 64, 64), "t64"),
                          ((32, 24, 16), "small"), ((40, 40, 24), "small"), ((37, 29, 21), "t4x4"),
                          ((30, 18, 7), "t2x2k1"), ((50, 47, 33), "t6x6k3"), ((130, 140, 72), "t16x16")]:
        a = rng.integers(-8, 9, size=(m, k), dtype=np.int64)
        b = rng.integers(-8, 9, size=(k, n), dtype=np.int64)
        for sch in all_schemes:
            add(f"int_{m}x{n}x{k}_{tl}_{sch.value}_clean", a, b, tl, sch, [], None)
            faults = [tiled.OutputFault(row=m // 3, col=n // 2, delta=7),
                      tiled.OutputFault(row=m - 1, col=0, delta=-3)]
            add(f"int_{m}x{n}x{k}_{tl}_{sch.value}_faults", a, b, tl, sch, faults, None)
    # thread-mma fault + canceling pair within one tile
    a = rng.integers(-8, 9, size=(64, 64), dtype=np.int64)
    b = rng.integers(-8, 9, size=(64, 64), dtype=np.int64)
    for sch in all_schemes:
        add(f"int_mma_{sch.value}", a, b, "t64", sch,
            [tiled.ThreadMmaFault(thread_row=2, thread_col=5, step=7, local_index=11, delta=3)], None)
        add(f"int_cancel_{sch.value}", a, b, "t64", sch,
            [tiled.OutputFault(row=1, col=1, delta=7), tiled.OutputFault(row=6, col=3, delta=-7)], None)
    # binary16 cases (tolerance parity): config 1 at 256^3 plus small ones
    for (m, n, k), tl in [((256, 256, 256), "default"), ((32, 24, 40), "small"), ((77, 90, 120), "t64"),
                          ((128, 128, 256), "t16x16")]:
        a = rng.uniform(-1, 1, size=(m, k)).astype(np.float16)
        b = rng.uniform(-1, 1, size=(k, n)).astype(np.float16)
        for sch in all_schemes:
            add(f"f16_{m}x{n}x{k}_{tl}_{sch.value}_clean", a, b, tl, sch, [], shapes.BINARY16)
            # one fault far above the responsible tau, one far below it
            faults = [tiled.OutputFault(row=3, col=5, delta=5000.0),
                      tiled.OutputFault(row=m - 2, col=n - 3, delta=1e-6)]
            add(f"f16_{m}x{n}x{k}_{tl}_{sch.value}_faults", a, b, tl, sch, faults, shapes.BINARY16)
    return cases


def make_pipeline_cases(checksum, shapes):
    rng = np.random.default_rng(77)
    cases = []
    for trial in range(24):
        exact = trial % 3 == 0
        depth = int(rng.integers(1, 5))
        batch = int(rng.integers(1, 9))
        dims = [int(rng.integers(4, 40)) for _ in range(depth + 1)]
        if exact:
            a0 = rng.integers(-5, 6, size=(batch, dims[0]), dtype=np.int64)
            ws = [rng.integers(-5, 6, size=(dims[j], dims[j + 1]), dtype=np.int64) for j in range(depth)]
            dtype = None
        else:
            a0 = rng.uniform(-0.5, 0.5, size=(batch, dims[0])).astype(np.float16)
            ws = [rng.uniform(-0.5, 0.5, size=(dims[j], dims[j + 1])).astype(np.float16) for j in range(depth)]
            dtype = shapes.BINARY16
        faults = {}
        if trial % 2 == 1:
            layer = int(rng.integers(depth))
            faults[layer] = [(int(rng.integers(batch)), int(rng.integers(dims[layer + 1])),
                              7.0 if exact else 1000.0)]
        checksum.clear_weight_checksum_cache()
        vs = checksum.run_protected_pipeline(a0, ws, dtype=dtype, faults=faults)
        meta = dict(name=f"pipe_{trial}", exact=exact, faults={str(k): v for k, v in faults.items()},
                    verdicts=[[bool(v.detected), float(v.lhs), float(v.rhs), float(v.tolerance_used)] for v in vs])
        arrays = {"a0": a0}
        for j, w in enumerate(ws):
            arrays[f"w{j}"] = w
        cases.append((meta, arrays))
    return cases


def make_select_cases(cost, shapes, tiled):
    T4 = shapes.DeviceProfile(name="T4", tensor_throughput=65e12, alu_throughput=65e12 / 8,
                              memory_bandwidth=320e9)
    B200 = shapes.DeviceProfile(name="B200", tensor_throughput=1670.1e12, alu_throughput=74e12,
                                memory_bandwidth=6372.2e9, verification_launch_latency=0.0)
    rng = np.random.default_rng(5)
    out = []
    for dev in (T4, B200):
        for s in (16, 32, 64, 128, 256, 512, 768, 1024, 1280, 2048, 4096):
            shape = shapes.GemmShape(s, s, s)
            out.append(dict(device=dev.name, kind="square", shape=[s, s, s],
                            base=cost.base_time(shape, shapes.BINARY16, dev),
                            times={sch.value: cost.scheme_time(shape, shapes.BINARY16, dev, sch)
                                   for sch in tiled.Scheme}))
        for trial in range(10):
            layers = [(i, shapes.GemmShape(*(8 * int(x) for x in rng.integers(1, 64, size=3))))
                      for i in range(int(rng.integers(1, 7)))]
            plan = cost.select(layers, shapes.BINARY16, dev)
            out.append(dict(device=dev.name, kind="plan",
                            layers=[[i, s.m, s.n, s.k] for i, s in layers],
                            chosen=[lp.chosen.value for lp in plan.layers],
                            agg_base=plan.aggregate_base_time, agg_prot=plan.aggregate_protected_time))
    return out


def make_campaign_cases(shapes, tiled):
    """Per-trial outcomes of the reference campaign (campaign.py:227-259) for parity of the
    GPU campaign: the trial draws (shape, delta, fault) and detected / masked / missed."""
    sys.path.insert(0, REF)
    from abft_guard import campaign as C
    out = []
    schemes = tuple(s for s in tiled.Scheme if s is not tiled.Scheme.UNPROTECTED)
    for dtype, delta, seed, ntr in ((shapes.EXACT_INT, C.INT_DELTAS, 20240601, 40),
                                    (shapes.BINARY16, C.FP_DELTAS, 7, 40)):
        cfg = C.CampaignConfig(trials=ntr, seed=seed, gemm_min=8, gemm_max=24, schemes=schemes, dtype=dtype,
                               delta=delta, control_trials=ntr)
        for si, sch in enumerate(schemes):
            for t in range(ntr):
                rng = C._trial_rng(seed, si, 0, t)
                shape = shapes.GemmShape(m=int(rng.integers(8, 25)), n=int(rng.integers(8, 25)),
                                        k=int(rng.integers(8, 25)))
                a, b = C.random_matrices(rng, shape, dtype)
                d = delta.sample(rng)
                site = C.SITE_OUTPUT if rng.integers(2) else C.SITE_THREAD_MMA
                f = (tiled.random_output_fault(rng, shape, d) if site == C.SITE_OUTPUT
                     else tiled.random_thread_mma_fault(rng, shape, cfg.tiling, d))
                rep = tiled.execute(a, b, cfg.tiling, sch, faults=[f], dtype=dtype)
                tau = C._fault_tolerance(rep, f, cfg.tiling)
                detected, masked = C._run_injected_trial(cfg, sch, si, t)
                outcome = "detected" if detected else ("masked" if masked else "missed")
                fdesc = (["output", f.row, f.col, float(f.delta)] if isinstance(f, tiled.OutputFault) else
                         ["thread-mma", f.thread_row, f.thread_col, f.step, f.local_index, float(f.delta)])
                out.append(dict(dtype=dtype.tag.value, seed=seed, scheme=sch.value, scheme_index=si, trial=t,
                                shape=[shape.m, shape.n, shape.k], delta=float(d), fault=fdesc,
                                outcome=outcome, tau=float(tau),
                                control_flagged=bool(C._run_control_trial(cfg, sch, si, t))))
    return out


def _save(cases, path):
    arrays, metas = {}, []
    for i, (meta, arrs) in enumerate(cases):
        metas.append(meta)
        for key, val in arrs.items():
            arrays[f"c{i}_{key}"] = val
    np.savez_compressed(path + ".npz", **arrays)
    with open(path + ".json", "w") as fh:
        json.dump(metas, fh, indent=0, sort_keys=True)


def main():
    checksum, cost, shapes, tiled = _ref()
    _save(make_execute_cases(tiled, shapes), os.path.join(HERE, "execute_cases"))
    _save(make_pipeline_cases(checksum, shapes), os.path.join(HERE, "pipeline_cases"))
    with open(os.path.join(HERE, "select_cases.json"), "w") as fh:
        json.dump(make_select_cases(cost, shapes, tiled), fh, indent=0, sort_keys=True)
    with open(os.path.join(HERE, "campaign_cases.json"), "w") as fh:
        json.dump(make_campaign_cases(shapes, tiled), fh, indent=0, sort_keys=True)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
