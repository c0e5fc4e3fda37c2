"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of every kernel in an
ncu --set full capture -> profiles/r01_traffic.json (mean over the captured launches of each kernel).
bench.py's roofline object reports it as `traffic` for its dominant kernel.
usage: python tools/make_traffic.py profiles/r01_full.ncu-rep [more.ncu-rep ...]"""
import csv, io, json, re, subprocess, sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(paths):
    out = {}
    for path in paths:
        raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        ki, a, b = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        acc = {}
        for r in rows[2:]:
            name = re.sub(r"\(.*", "", r[ki]).replace("<unnamed>::", "").replace("void ", "").strip()
            v = float(r[a]) * UNIT[units[a]] + float(r[b]) * UNIT[units[b]]
            acc.setdefault(name, []).append(v)
        for k, v in acc.items():
            out[k] = {"bytes_per_launch": sum(v) / len(v), "launches": len(v), "capture": path}
    json.dump(out, open("profiles/r01_traffic.json", "w"), indent=1, sort_keys=True)
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1:])
