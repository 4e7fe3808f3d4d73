"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

usage: python tools/ncu_summary.py <tag> <launches.csv> <kcell_metrics.csv> <full.ncu-rep> <stats.json>
"""
import collections, csv, json, subprocess, sys

tag, launches, kmet, rep, statsf = sys.argv[1:6]
out = {"tag": tag}

def rows_of(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    return [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "s": 1e6, "second": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(d):
    """metric value in us (times) or bytes (sizes)"""
    v = float(d["Metric Value"].replace(",", ""))
    return SCALE.get(d.get("Metric Unit", ""), 1.0) * v

# 1. launch list: share of each kernel in the device time of ONE solve (cold-cache,
# serialised).  The profiled command runs several solves (bench warm-up steps); the graph
# kernels of the round loop may be profiled for only some of them, so every kernel is
# normalised to one solve: per-round kernels (k_cell, k_select, k_round_end) by the rounds of
# a solve, once-per-solve kernels by their launch count.
stats = json.load(open(statsf))["stats"]
rounds = stats["rounds"]
PER_ROUND = ("k_cell", "k_select", "k_round_end")
agg = collections.defaultdict(lambda: [0, 0.0])
for d in rows_of(launches):
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("void ", "")
    agg[k][0] += 1
    agg[k][1] += val(d)
per_solve = {}
for k, (c, t) in agg.items():
    n_solve = rounds if k.startswith(PER_ROUND) else 1
    per_solve[k] = (t / c) * n_solve
tot = sum(per_solve.values())
out["launch_list"] = [{"kernel": k, "launches_profiled": agg[k][0], "us_per_launch": round(agg[k][1] / agg[k][0], 2),
                       "us_per_solve": round(t, 1), "share_of_solve": round(t / tot, 4)}
                      for k, t in sorted(per_solve.items(), key=lambda x: -x[1])]

# 2. k_cell DRAM traffic of the measured solve (the last `rounds` k_cell launches; the
# profiled command runs a warm-up solve first)
ids = collections.defaultdict(dict)
for d in rows_of(kmet):
    ids[int(d["ID"])][d["Metric Name"]] = val(d)
last = sorted(ids)[-max(rounds, 1):]   # async (rounds = 0): the one k_async launch
byts = collections.defaultdict(float)
for i in last:
    for m, v in ids[i].items():
        byts[m] += v
proc = stats["cell_processings"]
dram = byts.get("dram__bytes_read.sum", 0) + byts.get("dram__bytes_write.sum", 0)
out["kcell_traffic"] = {"dram_read": byts.get("dram__bytes_read.sum"), "dram_write": byts.get("dram__bytes_write.sum"),
                        "time_us": byts.get("gpu__time_duration.sum"), "launches": len(last), "processings": proc,
                        "dram_bytes_per_processing": dram / max(proc, 1),
                        "alg_bytes_per_processing": stats["bytes_cell_alg"] / max(proc, 1)}

# 3. one full capture of the top kernel
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hdr, row = rr[0], rr[2]
d = dict(zip(hdr, row))
units = dict(zip(hdr, rr[1]))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
out["full_capture"] = {k: (f"{d.get(k)} {units.get(k, '')}".strip() if d.get(k) is not None else None) for k in keys}
st = {k: float(d[k] or 0) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
tot = sum(st.values()) or 1
out["full_capture"]["stall_pct"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * v / tot, 1)
                                    for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]}
json.dump(out, open(f"profiles/r01_{tag}.json", "w"), indent=1)
print(json.dumps(out, indent=1))
