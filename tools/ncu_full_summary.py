"""Summarise `ncu --set full` reports (one block per captured launch) into a text file, and record
the DRAM bytes of the attention launches in profiles/attention_traffic.json (what bench.py reports as
roofline.traffic for the workload / input the capture was taken on).
usage: python tools/ncu_full_summary.py out.txt rep1.ncu-rep [rep2 ...]"""
import csv, io, json, os, subprocess, sys
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size']
HEADS, WORKLOAD, KIND = 8, "wan2.2-720p", "blobs"   # what tools/one_layer.py --heads 8 runs
att_bytes = 0.0
out = open(sys.argv[1], 'w')
out.write("ncu --set full --clock-control none --import-source on, tools/one_layer.py --heads 8 --calls 1\n"
          "(Wan2.2-720p shape, 8 of 40 heads, rho = 0.25); one block per captured launch\n")
for rep in sys.argv[2:]:
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d['Kernel Name'].split('(')[0].replace('void ', '')
        out.write(f"\n{name}   [{rep.split('/')[-1]}]\n")
        if 'attend_tc_kernel' in name:
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            for w in ('dram__bytes_read.sum', 'dram__bytes_write.sum'):
                att_bytes += float(d[w].replace(',', '')) * scale[units[hdr.index(w)]]
        for w in WANT:
            if w in d:
                out.write(f"    {w:72s} {d[w]} {units[hdr.index(w)]}\n")
out.close()
if att_bytes > 0:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "attention_traffic.json")
    rec = json.load(open(path)) if os.path.exists(path) else {}
    rec[f"{WORKLOAD}/{KIND}"] = {
        "dram_bytes": att_bytes, "heads": HEADS,
        "source": f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum of both attention launches, "
                  f"{HEADS}-head capture ({os.path.basename(sys.argv[1])}) scaled by heads"}
    json.dump(rec, open(path, "w"), indent=1)
