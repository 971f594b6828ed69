"""The reference's own training CLI (`python -m weightpack train`, default
config: 784-128-64-4 MLP, 2 workers, AWP on, 10 epochs) run twice on the GPU
box: once stock (baseline/_ref, NumPy codec) and once with its hot path
plugged (tests/refsuite/plug: weightpack.codec / weightpack.precision = this
package). Compares the run's own profile (profile.json phases: pack, unpack,
l2_norm wall seconds as the reference's PhaseTimer measures them) and checks
that the outputs that depend only on the weights — metrics.csv (losses,
accuracies), the ledger's byte columns and the trace's widths — are identical.

    python scripts/plugged_train_profile.py [--mode a2dtwp|baseline|oracle]
"""

import csv
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
STUBS = os.path.join(ROOT, "tests", "refsuite", "stubs")
PLUG = os.path.join(ROOT, "tests", "refsuite", "plug")


def run(plugged, cfg, out, mode, seed=1):
    env = dict(os.environ)
    if plugged:
        env["ADT_REFSUITE_REF"] = os.path.join(REF, "weightpack")
        env["PYTHONPATH"] = os.pathsep.join([PLUG, STUBS, ROOT])
    else:
        env["PYTHONPATH"] = os.pathsep.join([STUBS, REF])
    p = subprocess.run([sys.executable, "-m", "weightpack", "train", "--config", cfg, "--seed", str(seed),
                        "--out", out, "--mode", mode], env=env, capture_output=True, text=True, cwd=tempfile.gettempdir())
    if p.returncode != 0:
        raise RuntimeError(p.stdout + p.stderr)
    return p.stdout.strip().splitlines()[0]


def main():
    mode = sys.argv[sys.argv.index("--mode") + 1] if "--mode" in sys.argv else "a2dtwp"
    with tempfile.TemporaryDirectory() as tmp:
        cfg = os.path.join(tmp, "run.ini")
        env = dict(os.environ, PYTHONPATH=os.pathsep.join([STUBS, REF]))
        d = subprocess.run([sys.executable, "-m", "weightpack", "train", "--print-defaults"], env=env,
                           capture_output=True, text=True, check=True).stdout
        open(cfg, "w").write(d)
        outs = {}
        for name, plugged in (("stock", False), ("plugged", True)):
            out = os.path.join(tmp, name)
            summary = run(plugged, cfg, out, mode)
            prof = json.load(open(os.path.join(out, "profile.json")))
            outs[name] = (out, prof, summary)
            print(f"{name:8s} {summary}")
        print(json.dumps(outs["stock"][1])[:400])
        print(f"{'phase':10s} {'stock s':>10s} {'plugged s':>10s} {'ratio':>7s}")
        ps, pp = outs["stock"][1].get("phases", {}), outs["plugged"][1].get("phases", {})
        for ph in ps:
            a, b = ps[ph].get("wall_s", 0.0), pp.get(ph, {}).get("wall_s", 0.0)
            print(f"{ph:10s} {a:10.3f} {b:10.3f} {a / b if b else float('nan'):7.1f}x")
        same_metrics = open(os.path.join(outs["stock"][0], "metrics.csv")).read() == \
            open(os.path.join(outs["plugged"][0], "metrics.csv")).read()

        def ledger_bytes(o):
            rows = list(csv.DictReader(open(os.path.join(o, "ledger.csv"))))
            return [(r["batch"], r["direction"], r["layer"], r["raw_bytes"], r["wire_bytes"]) for r in rows]

        def widths(o):
            return [(r["batch"], r["layer"], r["bits"], r["counter"])
                    for r in csv.DictReader(open(os.path.join(o, "trace.csv")))]

        print("metrics.csv identical:", same_metrics)
        print("ledger byte columns identical:", ledger_bytes(outs["stock"][0]) == ledger_bytes(outs["plugged"][0]))
        print("trace widths/counters identical:", widths(outs["stock"][0]) == widths(outs["plugged"][0]))


if __name__ == "__main__":
    main()
