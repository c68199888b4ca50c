import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum','lts__t_sectors_srcunit_tex_op_read.sum','smsp__inst_executed.sum','sm__cycles_elapsed.avg','l1tex__throughput.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_lg.sum','l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active','l1tex__m_xbar2l1tex_read_sectors.sum', 'launch__grid_size',
        # L2 hit rates of the random Y gathers / reductions (north_star)
        'lts__t_sector_hit_rate.pct','lts__t_sector_op_read_hit_rate.pct','lts__t_sector_op_red_hit_rate.pct','lts__t_sector_op_atom_hit_rate.pct','lts__t_sectors_op_read.sum','lts__t_sectors_op_red.sum','lts__t_sectors_op_atom.sum','lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum','lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum']
for v in vals:
    print('---', v[hdr.index('Kernel Name')][:60] if 'Kernel Name' in hdr else '')
    for w in want:
        if w in hdr:
            i = hdr.index(w); print(f"  {w:70s} {units[i]:>10s} {v[i]}")
stall = [(h, v[hdr.index(h)]) for h in hdr if h.startswith('smsp__average_warp_latency_issue_stalled') or h.startswith('smsp__pcsamp_warps_issue_stalled')]
