"""Print the headline metrics of every kernel in an ncu report (ncu -i ... --page raw --csv)."""
import csv, subprocess, sys
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_write.sum',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed']
STALL = 'smsp__pcsamp_warps_issue_stalled_'
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print('==', r[hdr.index('Kernel Name')])
    for w in WANT:
        if w in hdr:
            print(f'  {w:70s} {r[hdr.index(w)]} {units[hdr.index(w)]}')
    st = sorted(((float(r[i] or 0), h[len(STALL):]) for i, h in enumerate(hdr)
                 if h.startswith(STALL) and not h.endswith('_not_issued')), reverse=True)[:8]
    print('  stalls (pc samples):', ', '.join(f'{n} {int(v)}' for v, n in st))
