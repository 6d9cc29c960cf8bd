"""The oracle (C restatement) pinned against the reference: committed golden
fixtures generated from the unmodified reference (tests/golden/make_golden.py),
the reference's own KATs, and — where the compiled reference is present — a
live field-by-field differential."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import simabi

GOLDEN = simabi.GOLDEN


def _fleet_goldens():
    with open(os.path.join(GOLDEN, "fleet_goldens.json")) as f:
        return json.load(f)["cases"]


def _bundled_trace(oracle_lib):
    # The bundled data/trace_zipf.csv equals the default synthetic trace
    # (proj/tests/test_trace.cpp:107-112); regenerate it with the oracle.
    f = oracle_lib.lib.orc_synthetic_trace_csv
    f.restype = C.c_void_p
    f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64]
    p = f(60, 6, 3000, 0.7063, 91)
    s = C.cast(p, C.c_char_p).value.decode()
    oracle_lib.lib.orc_free.argtypes = [C.c_void_p]
    oracle_lib.lib.orc_free(p)
    return s


@pytest.mark.parametrize("case", _fleet_goldens(),
                         ids=lambda c: f"g{c['gpus']}-ws{c['working_set']}-{c['policy']}-s{c['seed']}")
def test_oracle_matches_reference_goldens(oracle, table1, case):
    cfg = simabi.make_config(gpus=case["gpus"], working_set=case["working_set"], policy=case["policy"],
                             seed=case["seed"], o3_limit=case["o3_limit"], capacity_mb=case["capacity_mb"],
                             log_events=2, synthetic=False)
    res = oracle.run(table1, cfg, trace_csv=_bundled_trace(oracle))
    assert f"{res.decision_digest:016x}" == case["decision_digest"]
    assert f"{res.request_digest:016x}" == case["request_digest"]
    assert f"{res.log_digest:016x}" == case["log_digest"]
    for k, v in res.counts().items():
        assert v == case[k], k
    for k, v in case["report"].items():
        if k == "top_model":
            continue
        assert res.report[k] == v, k
    assert res.percentile_s(50) == case["p50_s"] and res.percentile_s(99) == case["p99_s"]


def test_survey_appendix_b1_counts(oracle, table1):
    """SURVEY.md Appendix B.1 decision/hit/miss/... counts (12 GPUs, ws 15, seed 1)."""
    want = {"lb": (1950, 520, 1430, 1238, 0, 1393, 0), "lalb": (2740, 1918, 32, 16, 790, 3, 0),
            "lalbo3": (2814, 1918, 32, 17, 864, 2, 7)}
    for pol, w in want.items():
        r = oracle.run(table1, simabi.make_config(gpus=12, policy=pol)).counts()
        got = (r["decisions"], r["hits"], r["misses"], r["false_misses"], r["local_enqueues"],
               r["evictions"], r["max_skip"])
        assert got == w, pol


def test_bundled_trace_generator(oracle):
    """Synthetic-trace KAT: totals and the 52-60% top-15 share (proj/tests/test_trace.cpp:80-95)."""
    csv = _bundled_trace(oracle).strip().splitlines()
    assert csv[0] == "function_id,m1,m2,m3,m4,m5,m6"
    rows = [list(map(int, line.split(",")[1:])) for line in csv[1:]]
    assert len(rows) == 60 and all(sum(r[m] for r in rows) == 3000 for m in range(6))
    tot = sorted((sum(r) for r in rows), reverse=True)
    share = sum(tot[:15]) / sum(tot)
    assert 0.52 <= share <= 0.60 and abs(share - 0.5611) < 5e-5  # "top-15 share 56.11%"


def test_mt19937_64_known_answer(oracle):
    """std::mt19937_64 KAT: the 10000th output for the default seed 5489 is
    9981545732273789042 (C++ standard [rand.predef])."""
    out = np.zeros(10000, dtype=np.uint64)
    oracle.lib.orc_mt19937_64.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
    oracle.lib.orc_mt19937_64(5489, 10000, out.ctypes.data)
    assert int(out[-1]) == 9981545732273789042


def test_oracle_vs_reference_live(oracle, ref, table1):
    for gpus in (1, 2, 3):
        for pol in ("lb", "lalb", "lalbo3"):
            for lim in ((0, 1, 25) if pol == "lalbo3" else (25,)):
                cfg = simabi.make_config(gpus=gpus, working_set=25, policy=pol, o3_limit=lim, seed=3,
                                         log_events=2)
                a, b = ref.run(table1, cfg), oracle.run(table1, cfg)
                simabi.assert_same(a, b, f"{gpus} {pol} {lim}")
                assert a.log_digest == b.log_digest


def test_oracle_mlp_catalog_goldens(oracle, mlp_catalog):
    path = os.path.join(GOLDEN, "mlp_c2_goldens.json")
    for case in json.load(open(path))["cases"]:
        cfg = simabi.make_config(gpus=case["gpus"], working_set=case["working_set"], policy=case["policy"],
                                 seed=case["seed"], o3_limit=case["o3_limit"], capacity_mb=case["capacity_mb"],
                                 log_events=2)
        res = oracle.run(mlp_catalog, cfg)
        assert f"{res.decision_digest:016x}" == case["decision_digest"]
        assert f"{res.log_digest:016x}" == case["log_digest"]


def test_oracle_errors(oracle, table1):
    with pytest.raises(simabi.SimError, match="cannot fit"):
        oracle.run(table1, simabi.make_config(capacity_mb=1000.0))
    with pytest.raises(simabi.SimError):
        oracle.run("model_id,occupation_mb,load_time_s,infer_time_s\n", simabi.make_config())
