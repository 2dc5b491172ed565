"""Summarize an ncu report: duration, pipe utilisation, DRAM, top stall SASS lines (dev tool)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
for data in rows[2:]:
    name = data[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(name[:90])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:70s} {data[i]:>16s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
out, h = [], None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        if h is not None: break
        continue
    if r and r[0] == "Address": h = r; continue
    if h and len(r) > 3:
        try: out.append((int(r[2]), r[1].strip()))
        except ValueError: pass
tot = max(1, sum(o[0] for o in out))
out.sort(reverse=True)
print("   top stall samples:")
for s, t in out[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"   {s:7d} {100*s/tot:5.1f}%  {t[:80]}")
