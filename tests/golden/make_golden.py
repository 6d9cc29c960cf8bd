"""Regenerates the committed golden fixtures from the UNMODIFIED reference.

Run HERE (needs /root/reference and oracle/_ref built by `make -C oracle ref`):
    python tests/golden/make_golden.py
Writes:
  tests/golden/table1_models.csv   paper Table I catalog (proj/data/models.csv, data only)
  tests/golden/trace_zipf.csv      bundled 60 x 6 invocation trace (proj/data/trace_zipf.csv, data only)
  tests/golden/fleet_goldens.json  per-config decision/request/log digests, counts,
                                   report fields and nearest-rank p50/p99 from the
                                   reference's run_stream
  tests/golden/mlp_c2_goldens.json the same for the B200 MLP catalog (configs[1])
The GPU box has no /root/reference, so tests there read only these files.
"""
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import simabi  # noqa: E402

REF_PROJ = "/root/reference/proj"


def record(res, cfg_desc):
    d = dict(cfg_desc)
    d.update(res.counts())
    d["decision_digest"] = f"{res.decision_digest:016x}"
    d["request_digest"] = f"{res.request_digest:016x}"
    d["log_digest"] = f"{res.log_digest:016x}"
    d["n_requests"] = int(len(res.arrival))
    d["p50_s"] = res.percentile_s(50)
    d["p99_s"] = res.percentile_s(99)
    d["report"] = {k: v for k, v in res.report.items() if k != "per_model"}
    return d


def fleet_cases():
    for gpus in (1, 12):
        for ws in (15, 25, 35):
            for pol in ("lb", "lalb", "lalbo3"):
                for seed in (1, 2):
                    yield dict(gpus=gpus, working_set=ws, policy=pol, seed=seed, o3_limit=25,
                               capacity_mb=8192.0)


def main():
    shutil.copyfile(os.path.join(REF_PROJ, "data", "models.csv"),
                    os.path.join(HERE, "table1_models.csv"))
    # bundled invocation trace (data only): the Azure-ingest round-trip test
    shutil.copyfile(os.path.join(REF_PROJ, "data", "trace_zipf.csv"),
                    os.path.join(HERE, "trace_zipf.csv"))
    ref = simabi.load_ref()
    cat = simabi.table1_catalog()
    trace = open(os.path.join(REF_PROJ, "data", "trace_zipf.csv")).read()
    out = []
    for case in fleet_cases():
        cfg = simabi.make_config(log_events=2, synthetic=False, **case)
        res = ref.run(cat, cfg, trace_csv=trace)
        out.append(record(res, case))
    with open(os.path.join(HERE, "fleet_goldens.json"), "w") as f:
        json.dump({"source": "oracle/_ref (unmodified reference run_stream), bundled trace_zipf.csv, "
                             "Table I catalog; log digest = FNV-1a-64 of EventLogger(dump_caches=true)",
                   "cases": out}, f, indent=1)
    mlp = os.path.join(os.path.dirname(HERE), "..", "paper_2303_05601_b200", "data", "mlp_c2_catalog.csv")
    if os.path.exists(mlp):
        mcat = open(mlp).read()
        out = []
        for pol in ("lb", "lalb", "lalbo3"):
            for seed in (1, 2, 3):
                case = dict(gpus=1, working_set=15, policy=pol, seed=seed, o3_limit=25, capacity_mb=204.0)
                cfg = simabi.make_config(log_events=2, **case)
                res = ref.run(mcat, cfg)
                out.append(record(res, case))
        with open(os.path.join(HERE, "mlp_c2_goldens.json"), "w") as f:
            json.dump({"source": "oracle/_ref run_stream on paper_2303_05601_b200/data/mlp_c2_catalog.csv",
                       "cases": out}, f, indent=1)
    print("wrote goldens")


if __name__ == "__main__":
    main()
