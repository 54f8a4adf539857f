"""Summarise an ncu report: key throughput metrics, stall reasons, DRAM bytes, smem wavefronts."""
import csv, subprocess, sys, io

def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    return rows

def main(rep):
    rows = raw(rep)
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v)); un = dict(zip(h, u))
        print("kernel:", d.get("Kernel Name", "")[:90])
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
                "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_alu.sum",
                "sm__inst_executed_pipe_xu.sum", "smsp__inst_executed_op_shared_ld.sum"]
        for k in keys:
            if k in d: print(f"  {k:70s} {d[k]:>18s} {un.get(k,'')}")
        st = []
        for k, val in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try: st.append((float(val), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError: pass
        tot = sum(x for x, _ in st) or 1
        print("  stalls:", ", ".join(f"{n} {x/tot*100:.0f}%" for x, n in sorted(st, reverse=True)[:8]))

if __name__ == "__main__":
    for r in sys.argv[1:]: main(r)
