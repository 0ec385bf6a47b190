"""Summarises ncu artefacts for profiles/: a launch list (--metrics gpu__time_duration.sum --csv)
and an `ncu --set full` report of one kernel.

  python tools/summarize_profiles.py launches.csv [full.ncu-rep] > SUMMARY.txt

Shares are of the solve's own kernels (rvb:: namespace); the live microbench peak kernel and
torch's L2-flush fill are listed but excluded from the shares.
"""
import collections
import csv
import subprocess
import sys

KEYS = ["SM Frequency", "Elapsed Cycles", "Duration", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Eligible Warps Per Scheduler", "Executed Instructions", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Branch Efficiency", "L1/TEX Hit Rate"]
RAW = ["smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
       "smsp__inst_executed_op_shared_atom.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0)))
    agg = collections.OrderedDict()
    for name, us in rows:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    own = sum(v[1] for k, v in agg.items() if "rvb::" in k)
    out = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
           "# share = of the solve's own kernels (rvb::); others listed without a share"]
    for name, (cnt, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = f"{100 * tot / own:6.1f}%" if "rvb::" in name and own else "       "
        out.append(f"{cnt:4d} launches  avg {tot / cnt:9.2f} us  {share}  {name[:100]}")
    return out


def full(path):
    out = [f"# ncu --set full: {path}"]
    res = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True)
    seen = set()
    for r in csv.DictReader(res.stdout.splitlines()):
        name = r.get("Metric Name")
        if name in KEYS and name not in seen:
            seen.add(name)
            out.append(f"{name} = {r['Metric Value']} {r['Metric Unit']}")
    res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(res.stdout.splitlines()))
    if len(rows) > 2:
        d = dict(zip(rows[0], rows[2]))
        u = dict(zip(rows[0], rows[1]))
        for k in RAW:
            if k in d:
                out.append(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
    return out


def kernel_json(path):
    """Per-launch numbers of the (single) kernel in an ncu --set full report, for bench.py."""
    res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(res.stdout.splitlines()))
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))

    def val(k, scale_units={"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6,
                            "usecond": 1e-3, "msecond": 1.0}):
        return float(d[k].replace(",", "")) * scale_units.get(u.get(k, ""), 1.0)

    return {"kernel": d["Kernel Name"], "source": path.split("/")[-1],
            "capture": "ncu --set full --clock-control none (one launch, cold cache, serialised)",
            "duration_ms": val("gpu__time_duration.sum"),
            "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "inst_executed": val("smsp__inst_executed.sum"),
            "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "shared_atom_inst": val("smsp__inst_executed_op_shared_atom.sum"),
            "shared_atom_wavefronts": val("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
            # the L1 data pipe (one wavefront per clock per SM): the vote's other co-binding limit
            # (peak 1 per clock per SM: wavefronts = pct x elapsed SM cycles x SMs)
            "lsu_wavefronts": val("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed") / 100.0
            * val("sm__cycles_elapsed.avg") * val("device__attribute_multiprocessor_count"),
            "lsu_wavefronts_pct": val("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            "shared_ld_wavefronts": val("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
            "sm_cycles": val("sm__cycles_elapsed.avg")}


def per_kernel(path):
    """One block per kernel launch of an ncu --set full report holding several kernels."""
    res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(res.stdout.splitlines()))
    if len(rows) < 3:
        return [f"# {path}: no launches"]
    h, u = rows[0], rows[1]
    keys = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
            ("dram__bytes_write.sum", "dram write"),
            ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
            ("launch__registers_per_thread", "registers/thread"), ("launch__grid_size", "grid"),
            ("launch__block_size", "block")]
    out = [f"# ncu --set full, one launch per kernel: {path}"]
    for r in rows[2:]:
        d = dict(zip(h, r))
        out.append(f"{d.get('Kernel Name', '?')[:110]}")
        for k, label in keys:
            if k in d:
                out.append(f"    {label:22s} {d[k]} {u[h.index(k)]}".rstrip())
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--kernels":
        print("\n".join(per_kernel(sys.argv[2])))
        sys.exit(0)
    if sys.argv[1] == "--json":
        import json
        print(json.dumps(kernel_json(sys.argv[2]), indent=1))
        sys.exit(0)
    lines = launches(sys.argv[1])
    if len(sys.argv) > 2:
        lines += [""] + full(sys.argv[2])
    print("\n".join(lines))
