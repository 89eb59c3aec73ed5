"""Record the DRAM traffic per launch of the timed pass kernel from an
`ncu --set full` capture into profiles/traffic.json (read by bench.py).
    python tools/traffic_json.py gpurun_out/prof_X.ncu-rep c2 fp64"""
import csv, io, json, os, subprocess, sys

rep, config, precision = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
row = next(r for r in data if "point_pass_hot" in r[hdr.index("Kernel Name")])
rd = float(row[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
wr = float(row[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
d = json.load(open(p)) if os.path.exists(p) else {}
d.setdefault(config, {})[precision] = {"dram_bytes": rd + wr, "read": rd, "write": wr,
                                       "kernel": row[hdr.index("Kernel Name")][:80],
                                       "source": os.path.basename(rep)}
json.dump(d, open(p, "w"), indent=1)
print(json.dumps(d[config][precision]))
