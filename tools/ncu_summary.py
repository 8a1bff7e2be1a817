"""Summarise ncu artefacts brought back in gpurun_out/ into small committed files under
profiles/: the per-kernel share of one step from a --metrics gpu__time_duration.sum launch
list, and the key metrics + top stall reasons of a --set full report.

  python tools/ncu_summary.py launches gpurun_out/X_launches.csv > profiles/..._launches.txt
  python tools/ncu_summary.py full gpurun_out/X.ncu-rep > profiles/..._ncu.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3}.get(r[ui], 1e-6)
        seq.append((r[ki].split("(")[0].replace("void ", "").split("<")[0].strip(), v * scale))
    starts = [i for i, (n, _) in enumerate(seq) if "k_subdiag" in n]
    last = seq[starts[-1]:] if starts else seq
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, v in last:
        tot[n] += v
        cnt[n] += 1
    T = sum(tot.values())
    out = ["# per-kernel device time of the last zz_tgevc call in the launch list (ncu, cold-cache,",
           "# serialised; compare shares, not absolutes).  source: %s" % path,
           "%-28s %8s %12s %8s" % ("kernel", "launches", "total ms", "share")]
    for n in sorted(tot, key=lambda n: -tot[n]):
        out.append("%-28s %8d %12.3f %7.2f%%" % (n, cnt[n], tot[n], 100 * tot[n] / T))
    out.append("%-28s %8d %12.3f" % ("TOTAL", sum(cnt.values()), T))
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = ["# ncu --set full summary.  source: %s" % path]
    for ridx, v in enumerate(rows[2:]):
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append("## launch %d: %s" % (ridx, name[:100]))
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append("  %-80s %s %s" % (k, v[i], u[i]))
        stalls = [(h[i], v[i]) for i in range(len(h))
                  if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("_per_issue_active.ratio")]
        stalls = sorted(((float(x), n) for n, x in stalls if x not in ("", "n/a")), reverse=True)[:8]
        out.append("  top stall reasons (warps per issue):")
        for x, n in stalls:
            out.append("    %-40s %.3f" % (n.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""), x))
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
