"""Summarise an ncu report: key metrics + per-source-line instruction/stall shares."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ("Duration", "Executed Ipc Active", "Issue Slots Busy", "DRAM Throughput", "Memory Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Theoretical Occupancy", "Compute (SM) Throughput")
seen = set()
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want and d["Metric Name"] not in seen:
        seen.add(d["Metric Name"])
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if len(rr) > 2:
    hh = rr[0]; vv = rr[2] if len(rr) > 2 else rr[1]
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "smsp__inst_executed_pipe_xu.sum"):
        if key in hh:
            print(f"{key:40s} {vv[hh.index(key)]} {rr[1][hh.index(key)]}")
    # warp stall breakdown (cycles per issued instruction, by reason)
    st = []
    for i, k in enumerate(hh):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(vv[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    if st:
        print("stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:10]))
    for key in ("smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed_op_shared_ld.sum",
                "smsp__inst_executed_op_shared_st.sum", "sm__sass_inst_executed_op_shared_ld.sum"):
        if key in hh:
            print(f"{key:40s} {vv[hh.index(key)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.Counter(); stall = collections.Counter(); txt = {}
cur = None; I = S = None
def num(x):
    try: return int(x)
    except Exception: return 0
for r in csv.reader(src.splitlines()):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No":
        I = r.index("Instructions Executed"); S = r.index("Warp Stall Sampling (All Samples)"); continue
    try: ln = int(r[0])
    except Exception: continue
    if I is not None and len(r) > I:
        agg[(cur, ln)] += num(r[I]); stall[(cur, ln)] += num(r[S]); txt[(cur, ln)] = r[1][:72]
tot = sum(agg.values()) or 1; st = sum(stall.values()) or 1
print("instructions", tot, "stall samples", st)
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1] / tot + stall[kv[0]] / st))[:top]:
    print(f"{100*v/tot:5.1f}% {100*stall[k]/st:5.1f}%  {k[0]}:{k[1]}  {txt[k]}")
