"""Pin the CPU oracle against the reference's own outputs (golden fixtures)."""

import numpy as np
import pytest

from oracle import abft_oracle as O


def _tiling(meta):
    f = meta["tiling_fields"]
    return O.Tiling(tb_m=f["tb_m"], tb_n=f["tb_n"], thread_m=f["thread_m"],
                    thread_n=f["thread_n"], k_step=f["k_step"])


def test_execute_matches_reference(execute_cases):
    assert len(execute_cases) >= 150
    for meta, arr in execute_cases:
        mode = "binary16" if meta["dtype"] == "binary16" else None
        faults = [tuple(f) for f in meta["faults"]]
        out, verdicts = O.execute(arr["a"], arr["b"], _tiling(meta), meta["scheme"], faults, mode)
        assert np.array_equal(out, arr["out"]), meta["name"]
        if meta["scheme"] == "global-abft":
            v = verdicts[0]
            assert [v.detected, v.lhs, v.rhs, v.tolerance_used] == meta["global"], meta["name"]
        else:
            got = np.array([[v.thread_row, v.thread_col, v.detected, v.max_abs_diff, v.tolerance_used]
                            for v in verdicts], dtype=np.float64).reshape(-1, 5)
            assert np.array_equal(got, arr["tv"]), meta["name"]
        assert any(v.detected for v in verdicts) == meta["detected"]
        tl = _tiling(meta)
        m, k = arr["a"].shape
        n = arr["b"].shape[1]
        assert list(O.op_counts(meta["scheme"], tl, m, n, k)) == meta["op_counts"], meta["name"]


def test_pipeline_matches_reference(pipeline_cases):
    for meta, arr in pipeline_cases:
        ws = [arr[f"w{j}"] for j in range(len(meta["verdicts"]))]
        faults = {int(k): [tuple(x) for x in v] for k, v in meta["faults"].items()}
        mode = None if meta["exact"] else "binary16"
        vs = O.pipeline(arr["a0"], ws, mode, faults)
        assert [[v.detected, v.lhs, v.rhs, v.tolerance_used] for v in vs] == meta["verdicts"], meta["name"]


def test_fig1_known_answers():
    # test_checksum.py:21-74 of the reference (Fig-1 toy)
    a = np.array([[1, 2], [3, 4]])
    b = np.array([[5, 6], [7, 8]])
    assert O.colck(a).tolist() == [4, 6]
    assert O.rowck(a).tolist() == [3, 7]
    assert O.dot(np.array([4, 6]), np.array([3, 7])) == 54
    c = O.matmul(a, b)
    assert c.tolist() == [[19, 22], [43, 50]] and O.total(c) == 134
    c2 = c.copy(); c2[0, 0] += 1; c2[1, 1] -= 1
    assert O.global_check(a, b, c2).detected is False       # canceling pair missed


def test_op_count_closed_forms():
    # test_tiled.py:261-271 of the reference (64^3, T64 tiling)
    t64 = O.Tiling(tb_m=64, tb_n=64, thread_m=16, thread_n=8, k_step=2)
    assert O.op_counts("thread-one-sided", t64, 64, 64, 64)[1] == 8192
    assert O.op_counts("thread-two-sided", t64, 64, 64, 64)[1] == 1024
    assert O.op_counts("thread-replication-full", t64, 64, 64, 64)[1] == 65536
    assert O.op_counts("global-abft", t64, 64, 64, 64)[2] == 64 * 64 + 64 + 64 * 64


def test_localization_known_answer():
    # test_tiled.py:106-112: ThreadMmaFault(2,5,step=7,local=11,delta=3) fires (2,5) only
    rng = np.random.default_rng(4)
    a = rng.integers(-8, 9, size=(64, 64), dtype=np.int64)
    b = rng.integers(-8, 9, size=(64, 64), dtype=np.int64)
    t64 = O.Tiling(tb_m=64, tb_n=64, thread_m=16, thread_n=8, k_step=2)
    _, vs = O.execute(a, b, t64, "thread-one-sided", [("thread-mma", 2, 5, 7, 11, 3)])
    assert [(v.thread_row, v.thread_col) for v in vs if v.detected] == [(2, 5)]


def test_im2col_matches_torch_unfold():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, size=(2, 9, 11, 5)).astype(np.float32)
    cols = O.im2col_nhwc(x, 3, 3, 2, 1)
    ref = torch.nn.functional.unfold(torch.from_numpy(x).permute(0, 3, 1, 2), 3, padding=1, stride=2)
    # unfold orders K as (c, r, s); ours is (r, s, c)
    ref = ref.view(2, 5, 3, 3, -1).permute(0, 4, 2, 3, 1).reshape(-1, 45).numpy()
    assert np.array_equal(cols, ref)
