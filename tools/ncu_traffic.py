"""Extract per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and duration
from `ncu --set full` reports into profiles/<round>/ncu_traffic.json (read by bench.py).

  python tools/ncu_traffic.py profiles/r01/ncu_traffic.json gpurun_out/r01e_*.ncu-rep
"""
import csv
import io
import json
import re
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    def get(name):
        i = h.index(name)
        return float(vals[i].replace(",", "")) * UNIT.get(units[i], 1.0)
    kname = vals[h.index("Kernel Name")]
    short = re.sub(r"^void |\(.*$", "", kname).replace("spc::", "")
    short = re.sub(r"<.*>", "", short).replace("_kernel", "")
    out = {"dram_bytes_read": get("dram__bytes_read.sum"), "dram_bytes_write": get("dram__bytes_write.sum"),
                   "traffic": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
                   "duration_ms_ncu": float(vals[h.index("gpu__time_duration.sum")].replace(",", "")) *
                   {"us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}.get(
                       units[h.index("gpu__time_duration.sum")], 1.0),
                   "report": rep.split("/")[-1]}
    # the shared-memory pipe (the binding resource of the scatter kernels): wavefronts per launch
    # and their share of the pipe's peak over the kernel's elapsed time
    for name, key in (("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared_wavefronts"),
                      ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                       "shared_pipe_pct_of_peak"),
                      ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared_bank_conflicts")):
        if name in h:
            try:
                out[key] = float(vals[h.index(name)].replace(",", ""))
            except ValueError:
                pass
    return short, out


if __name__ == "__main__":
    out = {}
    for rep in sys.argv[2:]:
        k, d = read(rep)
        out[k] = d
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1))
