"""DRAM traffic per launch of a kernel class from an ncu metrics CSV (dram__bytes_read/write.sum per launch):

    python tools/ncu_traffic.py gpurun_out/traffic.csv inner_gmres > profiles/r02_traffic.json

Writes {class: mean bytes per launch, ...detail} -- bench.py reads the class entry as roofline.traffic."""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_launches import load  # noqa: E402


def num(v):
    return float(v.replace(",", ""))


def main(path, cls):
    rows = load(path)
    tot, t_us, n = 0.0, 0.0, 0
    per = []
    for d in rows.values():
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if rd is None or wr is None:
            continue
        b = num(rd) + num(wr)
        # the capture uses --print-units base: bytes and nanoseconds
        per.append(b)
        tot += b
        t_us += num(d["gpu__time_duration.sum"]) / 1e3
        n += 1
    out = {cls: tot / max(n, 1), "launches": n, "total_bytes": tot, "total_ms": t_us / 1e3,
           "dram_gbs": tot / max(t_us, 1e-9) / 1e3,
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every inner_items_kernel launch "
                     "of one cfg5 64-RHS step (tools/r02_traffic.sh)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "inner_gmres")
