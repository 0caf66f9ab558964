"""Summarise ncu CSV exports into profiles/ (run in the build container).

  python tools/ncu_summary.py gpurun_out/launches_r1.csv gpurun_out/raw_g.csv gpurun_out/raw_f.csv \
      --out profiles/r1

Writes <out>_ncu_summary.md (per-kernel launch list shares of one timed step,
dram traffic per launch vs algorithmic bytes, key --set full metrics) and
<out>_traffic.json (dram bytes per launch, read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import json


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                           h.index("Metric Unit"), h.index("ID"))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0) * v  # -> us
        elif u in ("Kbyte", "KB"):
            v *= 1e3
        elif u in ("Mbyte", "MB"):
            v *= 1e6
        elif u in ("Gbyte", "GB"):
            v *= 1e9
        d = launches.setdefault(r[idi], {"name": r[ki].split("(")[0].replace("void ", "")})
        d[r[mi]] = v
    return list(launches.values())


UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def read_raw(path, want):
    """--page raw --csv export: row 0 names, row 1 units (which differ per column AND may
    differ from the unit another metric of the same family got: bytes are normalised to MB,
    durations to ms, so one column never mixes units)."""
    rows = list(csv.reader(open(path)))
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    out = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        rec = {"name": d.get("Kernel Name", "").split("(")[0]}
        for w in want:
            v, u = d.get(w, ""), units.get(w, "")
            if v != "" and u in UNIT and ("byte" in u or "second" in u):
                scale = UNIT[u] / (1e6 if "byte" in u else 1.0)
                v = f"{float(v.replace(',', '')) * scale:.3f}"
            rec[w] = v
        out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("launches")
    ap.add_argument("raw", nargs="*")
    ap.add_argument("--out", required=True)
    ap.add_argument("--steps", type=int, default=1, help="timed steps in the launch list")
    ap.add_argument("--last", type=int, default=0, help="keep only the last N launches")
    a = ap.parse_args()
    L = read_launches(a.launches)
    # bench.py --profile brackets the timed steps with cudaProfilerStart/Stop and ncu runs
    # with --profile-from-start off, so every listed launch belongs to the timed steps
    step = L[-a.last:] if a.last else L
    agg = collections.OrderedDict()
    for d in step:
        g = agg.setdefault(d["name"], {"n": 0, "us": 0.0, "dram": 0.0})
        g["n"] += 1
        g["us"] += d.get("gpu__time_duration.sum", 0.0)
        g["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    for g in agg.values():
        g["n_step"] = g["n"] / a.steps
    tot = sum(g["us"] for g in agg.values()) / a.steps
    lines = ["# ncu summary (one timed stage-solve, config 1, colour ordering)", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none` over `bench.py --steps 1 --warmup 1 --profile` (serialised, cold "
             "caches: compare shares, not absolute times).", "",
             f"Step total (serialised, per step over {a.steps} timed step(s)): {tot/1e3:.3f} ms", "",
             "| kernel | launches / step | time / step (ms) | share | DRAM bytes / launch (GB) |",
             "|---|---|---|---|---|"]
    for name, g in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        lines.append(f"| `{name}` | {g['n_step']:g} | {g['us']/1e3/a.steps:.3f} | {100*g['us']/a.steps/tot:.1f}% | "
                     f"{g['dram']/g['n']/1e9:.4f} |")
    # traffic per operation.  Per step: `it` Arnoldi products P^-1 (B v) (fused forward
    # launches + one backward sweep each), one plain apply (P^-1 b: forward + backward
    # sweeps), one plain matvec (true residual).  Backward sweeps: one launch per apply.
    import re

    def tot(pat):
        return sum(agg[n]["dram"] for n in agg if re.search(pat, n))

    def cnt(pat):
        return sum(agg[n]["n"] for n in agg if re.search(pat, n))
    it = cnt(r"k_multidot") or 1
    n_bwd = cnt(r"k_unc_sweep_seg<\d+, 0>|k_unc_bwd_pipe<\d+, \w+, false>") or 1
    bwd = tot(r"k_unc_sweep_seg<\d+, 0>|k_unc_bwd_pipe<\d+, \w+, false>") / n_bwd
    n_fused = it if cnt(r"k_unc_fused_fwd") else 0
    n_fwd = max(n_bwd - n_fused, 1)
    fwd = tot(r"k_copy_rows|k_unc_fwd_pipe|k_unc_bwd_pipe<\d+, \w+, true>|k_unc_sweep_seg<\d+, 1>") / n_fwd
    mv = [agg[n]["dram"] / agg[n]["n"] for n in agg if "k_stage_matvec" in n]
    traffic = {"stage_matvec": mv[0] if mv else None, "ilu0_apply": fwd + bwd}
    if n_fused:
        traffic["arnoldi_product"] = tot(r"k_unc_fused_fwd") / n_fused + bwd
    lines += ["", "DRAM traffic per operation (bytes):", "",
              f"* stage matvec: {traffic['stage_matvec']:.4e} (algorithmic 2.161e9)",
              f"* ILU apply (forward + backward sweeps of one apply): {traffic['ilu0_apply']:.4e} "
              f"(algorithmic 3.240e9 with the implicit-L factor)"]
    if n_fused:
        lines.append(f"* Arnoldi product P^-1 (B v) (fused forward + backward sweep): "
                     f"{traffic['arnoldi_product']:.4e} (algorithmic 4.709e9)")
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram__bytes_write.sum.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
    label = ["time (ms)", "DRAM read (MB)", "DRAM write (MB)", "DRAM read % of peak", "DRAM write % of peak",
             "issue slots busy %", "FP64/DMMA pipe busy % (pipe_shared)", "warps active %", "regs/thread",
             "stall short_scoreboard / issue", "stall long_scoreboard / issue", "stall barrier / issue",
             "stall math_pipe_throttle / issue"]
    for p in a.raw:
        lines += ["", f"## --set full metrics ({p.split('/')[-1]})", "",
                  "| kernel | " + " | ".join(label) + " |",
                  "|" + "---|" * (len(want) + 1)]
        for d in read_raw(p, want):
            lines.append(f"| `{d['name']}` | " + " | ".join(d[w] for w in want) + " |")
    open(a.out + "_ncu_summary.md", "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(a.out + "_traffic.json", "w"), indent=1)
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()
