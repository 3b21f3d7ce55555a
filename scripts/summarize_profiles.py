"""Turn the raw ncu artifacts a gpurun call brought back (gpurun_out/) into the committed
summaries under profiles/:  per-launch time list + per-kernel shares, the full-set metrics of
the dominant kernels, stall breakdowns, and profiles/switch_traffic.json (read by bench.py for
`roofline.traffic`).

    python scripts/summarize_profiles.py r01
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.max",
    "smsp__cycles_active.avg",
]


def ncu_csv(rep, page):
    res = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True)
    return list(csv.reader(res.stdout.splitlines()))


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    seq = []
    for row in rows:
        try:
            v = float(row["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            continue
        unit = row["Metric Unit"]
        v = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v * 1e6 if unit == "s" else v
        seq.append((row["Kernel Name"], v, row.get("Grid Size", ""), row.get("Block Size", "")))
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off  (AF_NCU=1 python bench.py --steps 3 --warmup 3)\n")
        f.write("# cold-cache, serialised launches of the e2e timed region: compare SHARES, not absolutes\n")
        f.write("index,kernel,duration_us,grid,block\n")
        for i, (k, v, g, b) in enumerate(seq):
            f.write(f'{i},"{k[:90]}",{v:.2f},"{g}","{b}"\n')
    agg = collections.defaultdict(list)
    for k, v, _, _ in seq:
        agg[k.split("(")[0][:60]].append(v)
    tot = sum(sum(v) for v in agg.values())
    with open(os.path.join(PROF, f"{tag}_launch_summary.txt"), "w") as f:
        f.write(f"{len(seq)} launches, {tot:.1f} us total (serialised under ncu)\n")
        f.write(f"{'kernel':62s} {'n':>5s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s}\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k:62s} {len(v):5d} {sum(v):10.1f} {sum(v) / len(v):9.2f} {sum(v) / tot:7.3f}\n")
    print(open(os.path.join(PROF, f"{tag}_launch_summary.txt")).read())


def full(tag, name, rep):
    rep = os.path.join(OUT, rep)
    if not os.path.exists(rep):
        return None
    raw = ncu_csv(rep, "raw")
    if len(raw) < 3:
        return None
    hdr, units = raw[0], raw[1]
    out = []
    first = None
    for row in raw[2:]:
        d = {h: (row[i], units[i]) for i, h in enumerate(hdr) if i < len(row)}
        if first is None:
            first = d
        out.append(f"--- {d.get('Kernel Name', ('?', ''))[0][:100]}")
        for k in KEYS:
            if k in d:
                out.append(f"    {k:80s} {d[k][0]:>16s} {d[k][1]}")
    src = ncu_csv(rep, "source")
    # stall breakdown of the first kernel
    blocks, cur = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    for b in blocks[:1]:
        hdr2 = b["rows"][0]
        data = [r for r in b["rows"][1:] if len(r) == len(hdr2)]
        idx = {h: i for i, h in enumerate(hdr2)}
        stalls = [h for h in hdr2 if h.startswith("stall_") and "Not Issued" not in h]
        tot = sum(int(r[idx["# Samples"]] or 0) for r in data) or 1
        out.append(f"\nwarp-state samples of {b['name'][:80]}: {tot}")
        agg = {s: sum(int(r[idx[s]] or 0) for r in data) for s in stalls}
        for s, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
            out.append(f"    {s:28s} {v:8d} {v / tot:6.3f}")
        out.append("top instructions by samples:")
        for r in sorted(data, key=lambda r: -int(r[idx["# Samples"]] or 0))[:12]:
            st = {s: int(r[idx[s]] or 0) for s in stalls}
            best = max(st.items(), key=lambda kv: kv[1])
            out.append(f"    {r[idx['# Samples']]:>7s}  {r[idx['Source']][:84]:84s} {best[0]}")
    with open(os.path.join(PROF, f"{tag}_{name}_full.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none --import-source on ; extracted with ncu -i ... --page raw/source --csv\n")
        f.write("\n".join(out) + "\n")
    return first


def to_bytes(first, key):
    v, u = first[key]
    v = float(v.replace(",", ""))
    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}.get(u, 1.0)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    chase = "--chase" in sys.argv   # artifacts of scripts/gpu_round4.sh (the one-pass schedule)
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    if chase:
        first = full(tag, "chase", "prof_chase.ncu-rep")
        if first:
            rd, wr = to_bytes(first, "dram__bytes_read.sum"), to_bytes(first, "dram__bytes_write.sum")
            layers = 32
            json.dump({"workload": "llama2-7b", "kernel": "switch_umma_kernel<4, GEMV> (one chained launch: o -> gate|up -> down -> next q|k|v)",
                       "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
                       "dram_bytes_per_token": (rd + wr) * layers,
                       "note": "a chained launch covers one layer's seven matrices; per token = per launch x 32 layers "
                               "(writes still in L2 at kernel end are not counted by dram__bytes_write)",
                       "source": f"profiles/{tag}_chase_full.txt (one ncu --set full capture inside bench.py's e2e region)"},
                      open(os.path.join(PROF, "chase_traffic.json"), "w"), indent=1)
            print("chase traffic per launch", (rd + wr) / 1e6, "MB")
        full(tag, "switch_umma", "prof_switch_umma.ncu-rep")
        full(tag, "tp_shard", "prof_shard.ncu-rep")      # one fused launch of a Llama-2-7B tp4 shard (partial tiles)
        for name, dst in (("chase_timeline.txt", "chase_timeline.txt"), ("umma_ab.txt", "umma_ab.txt"), ("umma_switch_ab.txt", "umma_switch_ab.txt"), ("bench.json", "bench.json"), ("bench_separate.json", "bench_separate.json"),
                          ("chase_kernel.txt", "chase_kernel.txt"), ("ab.txt", "consumer_loop_ab.txt")):
            pth = os.path.join(OUT, name)
            if os.path.exists(pth):
                with open(pth) as f, open(os.path.join(PROF, f"{tag}_{dst}"), "w") as g:
                    g.write(f.read())
        return
    first = full(tag, "switch", "prof_switch.ncu-rep")
    if first:
        rd, wr = to_bytes(first, "dram__bytes_read.sum"), to_bytes(first, "dram__bytes_write.sum")
        json.dump({"workload": "llama2-7b", "kernel": "switch_mma_kernel<2>", "dram_bytes_read": rd, "dram_bytes_write": wr,
                   "dram_bytes_per_launch": rd + wr, "source": f"profiles/{tag}_switch_full.txt (one ncu --set full capture, steady switch s=2kr)"},
                  open(os.path.join(PROF, "switch_traffic.json"), "w"), indent=1)
        print("switch traffic", (rd + wr) / 1e9, "GB")
    full(tag, "decode", "prof_gemv.ncu-rep")
    for name in ("tma_stream.log", "tile_stream.log", "sweep_variants.log", "bench_decode.log", "bench.json"):
        p = os.path.join(OUT, name)
        if os.path.exists(p):
            with open(p) as f, open(os.path.join(PROF, f"{tag}_{name.replace('.log', '.txt')}"), "w") as g:
                g.write(f.read())


if __name__ == "__main__":
    main()
