"""SURVEY.md s.8(d) oracle timing: the full oracle (oracle/, as it stands) on C2 (m = 2000) and
C3 (m = 10000) with all host cores and with one thread; prints one JSON object.
  python tools/oracle_time.py > profiles/<round>_oracle_time.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402

out = {"host_cores": os.cpu_count(), "runs": []}
try:
    out["cpu"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    pass
for name in ("C2", "C3"):
    S, T, _ = gen.config(name, seed=0)
    F = oracle.flops(S)
    for nth in (os.cpu_count(), 1):
        t0 = time.time()
        r = oracle.tgevc(S, T, nthreads=nth)
        dt = time.time() - t0
        assert r["status"] == 0
        out["runs"].append({"config": name, "m": S.shape[0], "threads": nth, "seconds": dt, "flops": F,
                            "gflops": F / dt * 1e-9})
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
