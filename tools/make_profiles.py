"""Turn the gpurun_out/ artifacts of tools/prof_round.sh into committed summaries:
profiles/<round>_launches.txt (kernel share of the step from the ncu launch list),
profiles/<round>_ncu_<kernel>.txt (ncu --set full summary), profiles/traffic.json (with the sha of the
library the captures are of: bench.py reports roofline.traffic only for that build)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(PROF, exist_ok=True)


def launches():
    path = os.path.join(OUT, "launches.csv")
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg, order = {}, []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        if k not in agg:
            order.append(k)
            agg[k] = [0, 0.0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
        agg[k][0] += 1
        agg[k][1] += ns
    setup = ("k_pubkey", "k_encrypt", "k_dlog_table", "k_decrypt")   # input generation, outside the timed step
    lib = {k: v for k, v in agg.items() if ("k_" in k) and not any(x in k for x in setup)}
    tot = sum(v[1] for v in lib.values()) or 1
    lines = [f"# ncu launch list ({rnd}): python bench.py --config c256 --steps 2 --warmup 1 "
             f"(--metrics gpu__time_duration.sum --clock-control none)",
             "# cold-cache, serialised launches: compare SHARES, not absolute times", "",
             f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k in order:
        if k in lib:
            n, ns = lib[k]
            lines.append(f"{k[:60]:60s} {n:8d} {ns / 1e6:10.3f} {100 * ns / tot:6.1f}%")
    open(os.path.join(PROF, f"{rnd}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def ncu_summary(rep, tag):
    if not os.path.exists(rep):
        return None
    s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                       text=True).stdout
    open(os.path.join(PROF, f"{rnd}_ncu_{tag}.txt"), "w").write(
        f"# ncu --set full --clock-control none, c256 bench, one launch ({rnd})\n" + s)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    d = dict(zip(rows[0], rows[2]))
    f = lambda k: float(d[k].replace(",", ""))
    u = dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = f("dram__bytes_read.sum") * scale.get(u["dram__bytes_read.sum"], 1)
    wr = f("dram__bytes_write.sum") * scale.get(u["dram__bytes_write.sum"], 1)
    print(s)
    return rd + wr


launches()
t_acc = ncu_summary(os.path.join(OUT, "prof_accum.ncu-rep"), "k_accum")
t_tab = ncu_summary(os.path.join(OUT, "prof_tables.ncu-rep"), "k_tables_coz")
tj = os.path.join(PROF, "traffic.json")
data = {}
sha = open(os.path.join(OUT, "lib_sha.txt")).read().strip() if os.path.exists(os.path.join(OUT, "lib_sha.txt")) else None
data["c256"] = {"lib_sha16": sha,
                "source": f"ncu --set full capture ({rnd}), dram__bytes_read.sum + dram__bytes_write.sum per launch"}
if t_acc:
    data["c256"]["accum_dram_bytes"] = t_acc
if t_tab:
    data["c256"]["tables_coz_dram_bytes"] = t_tab
json.dump(data, open(tj, "w"), indent=1)
