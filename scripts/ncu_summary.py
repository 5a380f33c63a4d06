"""Summarise ncu captures (gpurun_out/prof_<cfg>.ncu-rep, launches_<cfg>.csv) into
markdown rows: per kernel duration, DRAM bytes, DRAM throughput, tensor pipe,
occupancy.  Run here (no GPU needed)."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def main(cfgs):
    for c in cfgs:
        print(f"## {c}")
        for d in raw(f"gpurun_out/prof_{c}.ncu-rep"):
            name = d.get("Kernel Name", ("?", ""))[0][:40]
            vals = []
            for w in WANT:
                if w in d:
                    v, u = d[w]
                    vals.append(f"{w.split('__')[1].split('.')[0]}={v}{u}")
            print(f"- {name}: " + ", ".join(vals))
        try:
            rows = [r for r in csv.DictReader(l for l in open(f"gpurun_out/launches_{c}.csv") if l.startswith('"'))
                    if r.get("Metric Name")]
            by = {}
            for r in rows:
                by.setdefault((r["ID"], r["Kernel Name"][:30]), {})[r["Metric Name"]] = r["Metric Value"]
            print("  launch list (id, kernel, us, dram read MB, write MB):")
            for (i, k), m in list(by.items())[:8]:
                print(f"    {i} {k} {float(m.get('gpu__time_duration.sum', 0)) / 1e3:.2f} "
                      f"{float(m.get('dram__bytes_read.sum', 0)) / 1e6:.2f} {float(m.get('dram__bytes_write.sum', 0)) / 1e6:.2f}")
        except FileNotFoundError:
            pass


if __name__ == "__main__":
    main(sys.argv[1:] or ["few_shot"])
