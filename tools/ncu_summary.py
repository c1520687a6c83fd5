"""Summarise an ncu report (development aid): headline throughput metrics,
top stall reasons and a few counters per launch.

    python tools/ncu_summary.py report.ncu-rep [launch-id ...]
"""
import csv
import io
import subprocess
import sys

DETAILS = ["Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
           "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
           "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread", "Achieved Occupancy",
           "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "lts__t_requests_srcunit_tex.sum", "smsp__inst_executed.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct"]


def rows(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    want = set(sys.argv[2:])
    det = rows(rep, "details")
    hdr = det[0]
    ix = {h: i for i, h in enumerate(hdr)}
    seen = {}
    for r in det[1:]:
        lid = r[ix["ID"]]
        if want and lid not in want:
            continue
        if r[ix["Metric Name"]] in DETAILS:
            seen.setdefault(lid, {"kernel": r[ix["Kernel Name"]][:60]})[
                r[ix["Metric Name"]]] = f'{r[ix["Metric Value"]]} {r[ix["Metric Unit"]]}'
    raw = rows(rep, "raw")
    rh = raw[0]
    for r in raw[2:]:
        lid = r[rh.index("ID")]
        if want and lid not in want:
            continue
        d = seen.setdefault(lid, {})
        for k in RAW:
            if k in rh:
                d[k] = r[rh.index(k)]
        stalls = []
        for i, h in enumerate(rh):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[33:]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        d["top stalls"] = ", ".join(f"{n}={int(v)}" for v, n in stalls[:6])
    for lid, d in seen.items():
        print(f"== launch {lid}")
        for k, v in d.items():
            print(f"  {k:50s} {v}")


if __name__ == "__main__":
    main()
