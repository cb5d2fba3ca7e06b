"""Print the key metrics + top stall reasons + hottest SASS lines of an .ncu-rep."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Branch Efficiency", "No Eligible", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block", "Waves Per SM",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Frequency", "SM Frequency"]


KERNEL = []  # optional: --kernel-name regex:<argv[3]> (one kernel of a multi-kernel report)


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *KERNEL, *args], capture_output=True, text=True).stdout


def main(rep, nlines=25):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    seen = set()
    if rows:
        h = rows[0]
        iname, iunit, ival = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        for row in rows[1:]:
            if len(row) > ival and row[iname] in KEYS and row[iname] not in seen:
                seen.add(row[iname])
                print(f"{row[iname]:40s} {row[ival]:>14s} {row[iunit]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    if len(raw) > 2:
        h, v = raw[0], raw[2]
        for k, x in zip(h, v):
            if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                     "smsp__inst_executed.sum", "l1tex__t_bytes.sum"):
                print(f"{k:40s} {x:>14s} {raw[1][h.index(k)]}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv"))))
    at = next(i for i, r in enumerate(rows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r)
    hdr = rows[at]
    ci = hdr.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            float(x or 0)
            return True
        except ValueError:
            return False
    data = [r for r in rows[at + 1:] if len(r) == len(hdr) and num(r[ci])]
    ix = {c: i for i, c in enumerate(hdr)}
    col = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r[ix[col]] or 0) for r in data) or 1.0
    stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    agg = {s: sum(float(r[ix[s]] or 0) for r in data) for s in stalls}
    print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in
                               sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for r in sorted(data, key=lambda r: -float(r[ix[col]] or 0))[:nlines]:
        smp = float(r[ix[col]] or 0)
        st = sorted(((float(r[ix[s]] or 0), s) for s in stalls), reverse=True)[0]
        print(f"{100 * smp / tot:5.2f}% thr={r[ix['Avg. Threads Executed']]:>5} "
              f"{r[ix['Source']][:58]:58s} {st[1][6:]}")


if __name__ == "__main__":
    if len(sys.argv) > 3:
        KERNEL[:] = ["--kernel-name", "regex:" + sys.argv[3]]
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
