"""Regenerate profiles/<tag>_ncu_full.md, profiles/<tag>_launches.md and
profiles/traffic.json from the ncu outputs of scripts/ncu_r02c.sh in
gpurun_out/ (and copy the bench lines gpurun_out/<tag>_bench*.json).

    python scripts/profiles_summary.py [tag]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02c"
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    """[(kernel, us, dram bytes)] per launch of an ncu --metrics CSV."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    by = {}
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").replace("pmf::", "")
        e = by.setdefault(r[0], [name, 0.0, 0.0])
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        if r[mi] == "gpu__time_duration.sum":
            e[1] += v
        elif r[mi].startswith("dram"):
            e[2] += v
    return [tuple(v) for _, v in sorted(by.items(), key=lambda kv: int(kv[0]))]


def per_kernel(seq, prefix):
    sel = [(us, b) for k, us, b in seq if k == prefix or k.startswith(prefix + "<")]
    return (sum(b for _, b in sel) / max(1, len(sel)), len(sel), sum(us for us, _ in sel))


# ---- launch lists
lt = [f"# {TAG} launch lists (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
      "dram__bytes_write.sum --clock-control none; cold caches, serialised launches: the SHARES are "
      "what compares with the bench, not the absolute times)\n",
      f"Command: scripts/ncu_r02c.sh {TAG} (scripts/probe.py; step-synchronous batches with --graph 0 so "
      "every kernel is a separate launch).\n"]
lists = {}
for f, desc in (("c5", "C5 batch: 32 CPMC images (rng_seed 0..31), host-staged planes, step-synchronous"),
                ("c5s", "C5 batch: the same 32 images, planes derived on the device (pmf_synth_stage)"),
                ("c3", "C3: one CPMC image (rng_seed 0), asynchronous solver"),
                ("c2", "C2: 500x375, 20 lambdas, asynchronous solver")):
    path = os.path.join(G, f"{TAG}_launches_{f}.csv")
    if not os.path.exists(path):
        continue
    seq = launches(path)
    lists[f] = seq
    tot = {}
    for k, us, b in seq:
        t = tot.setdefault(k, [0, 0.0, 0.0])
        t[0] += 1
        t[1] += us
        t[2] += b
    T = sum(v[1] for v in tot.values())
    lt.append(f"## {desc}\n\n{len(seq)} launches, {T / 1e3:.3f} ms of kernel time\n")
    lt.append("| kernel | launches | total ms | share | avg us | DRAM MB / launch | DRAM GB/s |")
    lt.append("|---|---|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k][1]):
        n, us, b = tot[k]
        lt.append(f"| {k} | {n} | {us / 1e3:.3f} | {100 * us / T:.1f}% | {us / n:.1f} | {b / n / 1e6:.2f} | "
                  f"{b / us / 1e3 if us else 0:.0f} |")
    lt.append("")
open(os.path.join(P, f"{TAG}_launches.md"), "w").write("\n".join(lt) + "\n")

# ---- traffic.json (read by bench.py for roofline.traffic)
out = {}
for f, k, desc in (("c2", "k_async", "C2 (500x375, 20 lambdas, one supergraph)"),
                   ("c3", "k_async", "C3 (one CPMC image, 1000 lambda-graphs)"),
                   ("c5", "k_push", "C5 batch (32 images, step-synchronous mode)")):
    if f in lists:
        b, n, _ = per_kernel(lists[f], k)
        out.setdefault(k, {})[f] = {"dram_bytes_per_launch": b, "launches": n, "workload": desc}
if out:
    res = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     f"--clock-control none (scripts/ncu_r02c.sh {TAG}); cold-cache, serialised"}
    for k, v in out.items():
        first = next(iter(v.values()))
        res[k] = dict(first, per_config=v)
    json.dump(res, open(os.path.join(P, "traffic.json"), "w"), indent=1)

# ---- --set full captures
keys = ('Duration', 'Elapsed Cycles', 'Executed Instructions', 'Executed Ipc Active', 'Issue Slots Busy',
        'Warp Cycles Per Issued Instruction', 'Achieved Occupancy', 'Registers Per Thread',
        'Static Shared Memory Per Block', 'Block Size', 'Grid Size', 'DRAM Throughput', 'Memory Throughput',
        'L2 Hit Rate', 'L1/TEX Hit Rate', 'Avg. Active Threads Per Warp', 'Branch Efficiency')
lines = [f"# {TAG} ncu --set full captures (--clock-control none --import-source on)\n",
         f"Command: scripts/ncu_r02c.sh {TAG}.  `k_push` = tile discharge of the step-synchronous mode "
         "(C5), `k_bfs_sink` = exact global relabel, `k_async` = the asynchronous solve kernel (one launch "
         "solves the batch, C2/C3), `k_synth_*` / `k_pack_bits` = on-device synthesis and output packing "
         "(plain streaming kernels: their DRAM throughput is the HBM roofline).\n"]
for f, desc in ((f"{TAG}_k_push_c5", "k_push (9th launch), C5 batch of 32 images"),
                (f"{TAG}_k_bfs_c5", "k_bfs_sink (41st launch), C5 batch of 32 images"),
                (f"{TAG}_k_async_c3", "k_async, C3 (one CPMC image: 50 warm-start chains x 20 lambdas)"),
                (f"{TAG}_k_synth_c5", "on-device synthesis + packing, C5 batch of 32 images")):
    rep = os.path.join(G, f + ".ncu-rep")
    if not os.path.exists(rep):
        continue
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(det.splitlines()))
    h = r[0]
    per = {}
    for row in r[1:]:
        d = dict(zip(h, row))
        kn = d["Kernel Name"].split("(")[0].replace("void ", "").replace("pmf::", "")
        vals = per.setdefault((d["ID"], kn), {})
        if d['Metric Name'] in keys and d['Metric Name'] not in vals:
            vals[d['Metric Name']] = d['Metric Value'] + ' ' + d['Metric Unit']
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    for (kid, kn), vals in per.items():
        lines.append(f"## {desc}: `{kn}`\n\n| metric | value |\n|---|---|")
        lines += [f"| {k} | {vals[k]} |" for k in keys if k in vals]
        row = next((x for x in rr[2:] if x and x[0] == kid), None)
        if row:
            d = dict(zip(rr[0], row))
            try:
                b = sum(float(d[m].replace(",", "")) * SCALE.get(rr[1][rr[0].index(m)], 1)
                        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                lines.append(f"| dram bytes (read + write) | {b / 1e6:.3f} MB |")
            except (KeyError, ValueError):
                pass
            st = {}
            for k, x in d.items():
                if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                    try:
                        st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(x.replace(",", ""))
                    except ValueError:
                        pass
            tot = sum(st.values())
            if tot:
                lines.append("\nWarp stall samples (share):\n")
                lines += [f"- {k}: {100 * x / tot:.1f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:8]]
        lines.append("")
open(os.path.join(P, f"{TAG}_ncu_full.md"), "w").write("\n".join(lines) + "\n")

# ---- bench lines
for src in sorted(os.listdir(G)):
    if src.startswith(f"{TAG}_bench") and src.endswith(".json"):
        with open(os.path.join(G, src)) as fh:
            last = [ln for ln in fh.read().splitlines() if ln.startswith("{")]
        if last:
            with open(os.path.join(P, src), "w") as fh:
                fh.write(last[-1] + "\n")
print("ok")
