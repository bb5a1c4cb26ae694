"""From an `ncu --set full` report, write the measured DRAM traffic per launch
(dram__bytes_read.sum + dram__bytes_write.sum, averaged over the captured
launches of each kernel family) to profiles/traffic.json, which bench.py
reports as roofline.traffic.   python tools/ncu_traffic.py REPORT [OUT]"""
import csv
import io
import json
import subprocess
import sys

FAMILIES = {"k_gemm_tc": "gemm_tc", "k_fcgscan": "fcgscan", "k_quant": "quant", "k_scan": "scan",
            "k_gemv": "gemv"}


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
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
               "source": f"ncu --set full ({rep.split('/')[-1]})"} for k, v in acc.items()}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
