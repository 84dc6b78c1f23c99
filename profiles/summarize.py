"""Summarise ncu captures (run here, on the CPU box, from gpurun_out/ files).

    python profiles/summarize.py launches gpurun_out/launches_r1.csv > profiles/r1_launches.md
    python profiles/summarize.py full gpurun_out/prof_r1_exact.ncu-rep > profiles/r1_exact_ncu.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    i_name, i_val = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[i_name].split("(")[0].split("<")[0]
        tot[name] += float(r[i_val].replace(",", ""))
        cnt[name] += 1
    all_t = sum(tot.values())
    print("| kernel | launches | total time | share |")
    print("|---|---|---|---|")
    for k, t in tot.most_common():
        print(f"| {k} | {cnt[k]} | {t:.0f} | {t / all_t * 100:.1f}% |")


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    seen = set()
    for v in r[2:]:  # the first captured launch of every kernel
        name = v[h.index('Kernel Name')]
        if name in seen:
            continue
        seen.add(name)
        print(f"kernel: {name[:120]}")
        print("| metric | value | unit |")
        print("|---|---|---|")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {k} | {v[i]} | {u[i]} |")
        st = [(n, float(v[i])) for i, n in enumerate(h)
              if n.startswith("smsp__average_warps_issue_stalled")
              and n.endswith("per_issue_active.ratio") and v[i] not in ("", "n/a")]
        print("\nwarp stall reasons (per issued instruction):")
        for n, x in sorted(st, key=lambda t: -t[1])[:8]:
            print(f"- {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {x:.2f}")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
