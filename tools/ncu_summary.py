"""Summarise an ncu --set full capture into profiles/<name>.md (key raw metrics +
the top source lines by stall samples)."""
import csv, io, subprocess, sys, json
rep, name, title = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x"]
out = {}
lines = [f"# {title}", "", f"Capture: `{rep.split('/')[-1]}` (ncu --set full --clock-control none --import-source on; one launch).", "",
         "| metric | value | unit |", "|---|---|---|"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        out[w] = vals[i]
        lines.append(f"| {w} | {vals[i]} | {units[i]} |")
src = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "15"], capture_output=True, text=True).stdout
lines += ["", "Top source lines by warp-stall samples (tools/ncu_lines.py):", "", "```", src.rstrip(), "```", ""]
open(f"profiles/{name}.md", "w").write("\n".join(lines))
print("\n".join(lines[:20]))
json.dump(out, open(f"profiles/{name}.json", "w"), indent=1)
