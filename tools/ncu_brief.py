"""One-screen brief of an ncu --set full report: duration, DRAM / L2 traffic and
throughput, tensor / FP64 pipe activity, shared-memory wavefronts, occupancy,
issue activity and the top warp-stall reasons.

    python tools/ncu_brief.py report.ncu-rep [...]  > brief.txt
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes (all requests)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (realtime)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tc.sum", "tc pipe instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]


def main(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        if len(rows) < 3:
            print(p, "no data")
            continue
        hdr = rows[0]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            print(f"== {p}: {d.get('Kernel Name', '?')[:90]}")
            for k, name in KEYS:
                if k in d:
                    print(f"   {name:34s} {d[k]}")
            stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled_")
                      or k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
            vals = []
            for k, v in stalls:
                try:
                    vals.append((float(v.replace(",", "")), k))
                except ValueError:
                    pass
            vals.sort(reverse=True)
            tot = sum(v for v, _ in vals if "pcsamp" in _) or 1.0
            top = [(v, k) for v, k in vals if "pcsamp" in k][:6]
            if top:
                print("   top stall samples: " + ", ".join(
                    f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for v, k in top))


if __name__ == "__main__":
    main(sys.argv[1:])
