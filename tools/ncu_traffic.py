"""From an `ncu --set full` report, write the measured DRAM traffic per launch
(dram__bytes_read.sum + dram__bytes_write.sum, averaged over the captured
launches of each kernel family) to profiles/traffic.json under the config's key, which
bench.py reports as roofline.traffic for that config.
python tools/ncu_traffic.py REPORT --config c2 [--desc "what was captured"]"""
import csv
import io
import json
import subprocess
import sys

FAMILIES = {"k_gemm_tc": "gemm_tc", "k_gemm_2sm": "gemm_tc", "k_fcgscan": "fcgscan",
            "k_quant": "quant", "k_scan": "scan", "k_gemv": "gemv"}


def main():
    rep = sys.argv[1]
    cfg = sys.argv[sys.argv.index("--config") + 1]
    desc = sys.argv[sys.argv.index("--desc") + 1] if "--desc" in sys.argv else ""
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else "profiles/traffic.json"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = {}
    for r in rows[2:]:
        fam = next((v for k, v in FAMILIES.items() if k in r[idx["Kernel Name"]]), None)
        if fam is None:
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[idx[m]].replace(",", "")) * scale.get(units[idx[m]], 1)
        acc.setdefault(fam, []).append(tot)
    res = {k: {"bytes_per_launch": round(sum(v) / len(v)), "launches": len(v),
               "source": f"ncu --set full ({rep.split('/')[-1]})", "config": desc}
           for k, v in acc.items()}
    try:
        db = json.load(open(out))
    except Exception:
        db = {}
    db.setdefault(cfg, {}).update(res)
    json.dump(db, open(out, "w"), indent=1)
    print(json.dumps({cfg: res}, indent=1))


if __name__ == "__main__":
    main()
