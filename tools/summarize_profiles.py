"""Summarise a round's ncu output (launch lists + one full capture per config) into profiles/<round>/.

python tools/summarize_profiles.py gpurun_out/final profiles/r01
Writes ncu_<cfg>_summary.txt (key counters of the group-GEMM + kernel shares of the step from the
launch list) and profiles/ncu_traffic_<cfg>.json (dram bytes per launch, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def launches(path):
    lines = open(path).read().splitlines()
    i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(lines[i:]):
        k = r["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"]) / 1e3
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    for cfg in ("dsv2", "q15", "mx", "q2"):
        rep = os.path.join(src, f"prof_{cfg}.ncu-rep")
        lf = os.path.join(src, f"launches_{cfg}.csv")
        if not os.path.exists(rep):
            continue
        m = raw(rep)
        lines = [f"# ncu --set full --clock-control none -k regex:moe_gemm -s 2 -c 1: python bench.py --config {cfg} "
                 f"--steps 1 --warmup 2 (one moe_gemm_kernel launch)"]
        for k in KEYS:
            if k in m:
                lines.append(f"{k:70s} {m[k][0]:>18s} {m[k][1]}")
        if os.path.exists(lf):
            agg = launches(lf)
            tot = sum(t for _, t in agg.values())
            lines.append(f"# launch list (ncu --metrics gpu__time_duration.sum, {sum(n for n, _ in agg.values())} "
                         "launches, cold-cache serialised): share of the step per kernel")
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
                lines.append(f"{k:40s} launches {n:4d}  avg {t / n:9.1f} us  share {100 * t / tot:5.1f} %")
        open(os.path.join(dst, f"ncu_{cfg}_summary.txt"), "w").write("\n".join(lines) + "\n")

        def num(k):
            v, u = m[k]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        # tagged with the library it was captured on (the capture must come from this tree's libmxmoe.so):
        # bench.py reports roofline.traffic only for the same library build and token count
        import hashlib
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from synth import configs as C
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2505_05799_b200",
                               "libmxmoe.so"), "rb") as f:
            sha = hashlib.sha1(f.read()).hexdigest()
        json.dump({"kernel": "moe_gemm_kernel", "config": f"{cfg} mixed (bench default tokens)",
                   "tokens": C.get_config(cfg).tokens, "lib_sha1": sha,
                   "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                   "source": os.path.join(dst, f"ncu_{cfg}_summary.txt")},
                  open(os.path.join(os.path.dirname(dst.rstrip("/")), f"ncu_traffic_{cfg}.json"), "w"), indent=1)
        print(open(os.path.join(dst, f"ncu_{cfg}_summary.txt")).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
