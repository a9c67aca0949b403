"""Summarise `ncu --set full` reports (one block per captured launch) into a text file.
usage: python tools/ncu_full_summary.py out.txt rep1.ncu-rep [rep2 ...]"""
import csv, io, subprocess, sys
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
        for w in WANT:
            if w in d:
                out.write(f"    {w:72s} {d[w]} {units[hdr.index(w)]}\n")
out.close()
