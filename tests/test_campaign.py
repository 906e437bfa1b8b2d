"""Fault-injection campaign parity (the reference's campaign semantics, campaign.py:198-259).

CPU: the seeded trial generator (shape, operands, delta, site, fault position) equals the
reference's draw for draw.  GPU: every injected trial run on the sm_100a path has the
reference's outcome (detected / masked / missed) — bit-exact in exact-int mode; in binary16
a differing outcome is only allowed for a fault within [0.5 tau, 2 tau] of the responsible
verdict (fp32 summation order) — and no fault-free control trial is flagged.
"""

import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cases():
    with open(os.path.join(ROOT, "tests", "golden", "campaign_cases.json")) as fh:
        return json.load(fh)


def _config(P, C, case):
    dtype = P.EXACT_INT if case["dtype"] == "exact-int" else P.BINARY16
    delta = C.INT_DELTAS if dtype.is_exact else C.FP_DELTAS
    schemes = tuple(s for s in P.Scheme if s is not P.Scheme.UNPROTECTED)
    return C.CampaignConfig(trials=40, seed=case["seed"], gemm_min=8, gemm_max=24, schemes=schemes, dtype=dtype,
                            delta=delta, control_trials=40)


def test_trial_generator_matches_reference():
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import campaign as C
    cases = _cases()
    assert len(cases) == 400
    for case in cases:
        cfg = _config(P, C, case)
        shape, a, b, delta, fault = C.trial_spec(cfg, case["scheme_index"], case["trial"])
        assert [shape.m, shape.n, shape.k] == case["shape"]
        assert delta == case["delta"]
        if case["fault"][0] == "output":
            assert isinstance(fault, P.OutputFault)
            assert [fault.row, fault.col, fault.delta] == case["fault"][1:]
        else:
            assert isinstance(fault, P.ThreadMmaFault)
            assert [fault.thread_row, fault.thread_col, fault.step, fault.local_index, fault.delta] == \
                case["fault"][1:]


@pytest.mark.gpu
def test_campaign_outcomes_match_reference():
    import paper_2104_09455_b200 as P
    from paper_2104_09455_b200 import campaign as C, device
    device.require_device()
    mismatches = []
    for case in _cases():
        cfg = _config(P, C, case)
        scheme = P.Scheme(case["scheme"])
        outcome, delta, tau = C.injected_trial(cfg, scheme, case["scheme_index"], case["trial"])
        if outcome != case["outcome"]:
            near = 0.5 * case["tau"] <= abs(case["delta"]) <= 2.0 * case["tau"]
            if case["dtype"] == "exact-int" or not near:
                mismatches.append((case["dtype"], case["scheme"], case["trial"], outcome, case["outcome"],
                                   delta, tau, case["tau"]))
        assert C.control_trial(cfg, scheme, case["scheme_index"], case["trial"]) is case["control_flagged"] is False
    assert not mismatches, mismatches[:10]
