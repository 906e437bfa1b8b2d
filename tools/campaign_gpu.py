"""Fault-injection campaign at scale on the sm_100a path (campaign.py semantics).

Every injected trial is one seeded GEMM with one fault (output element or thread-MMA operand)
executed through the drop-in ``execute``; a trial is detected / masked-by-tolerance / missed as
in campaign.py:213-247; fault-free control trials count false positives.
usage: python tools/campaign_gpu.py [--trials N] [--out FILE]"""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--out", default="gpurun_out/campaign_gpu.json")
    args = ap.parse_args()
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import campaign as C
    schemes = tuple(s for s in P.Scheme if s is not P.Scheme.UNPROTECTED)
    res = {"trials_per_scheme": args.trials, "control_trials_per_scheme": args.trials, "configs": []}
    for (dname, dtype, delta), site in itertools.product(
            (("exact-int", P.EXACT_INT, C.INT_DELTAS), ("binary16", P.BINARY16, C.FP_DELTAS)),
            (C.SITE_OUTPUT, C.SITE_THREAD_MMA)):
        cfg = C.CampaignConfig(trials=args.trials, seed=2104, gemm_min=8, gemm_max=96, schemes=schemes, dtype=dtype,
                               delta=delta, control_trials=args.trials, site=site)
        t0 = time.time()
        stats = C.run_campaign(cfg)
        row = {"dtype": dname, "site": site, "gemm_extent": [8, 96],
               "deltas": f"{delta.kind} [{delta.low}, {delta.high}]",
               "wall_s": round(time.time() - t0, 1), "schemes": {}}
        for s, st in stats.items():
            row["schemes"][s.value] = dict(injected=st.injected_trials, detected=st.detected,
                                           masked_by_tolerance=st.masked_by_tolerance, missed=st.missed,
                                           detection_rate_of_unmasked=(st.detected / max(1, st.detected + st.missed)),
                                           control=st.control_trials, false_positives=st.false_positives)
        res["configs"].append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
