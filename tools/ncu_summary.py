import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
keep = ['Duration','DRAM Throughput','L1/TEX Cache Throughput','Compute (SM) Throughput','SM Active Cycles','Elapsed Cycles','Issue Slots Busy','Achieved Occupancy','Registers Per Thread','Dynamic Shared Memory Per Block','Grid Size','Block Size','Theoretical Occupancy','Warp Cycles Per Issued Instruction','Eligible Warps Per Scheduler','Executed Instructions','Memory Throughput','L2 Hit Rate']
for row in r[1:]:
    d = dict(zip(hdr, row))
    if d.get('Metric Name') in keep:
        print(d['Kernel Name'][:20], d['Metric Name'].ljust(40), d['Metric Unit'].ljust(10), d['Metric Value'])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, units = r[0], r[1]
want = ['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','l1tex__throughput.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum']
want += [h for h in hdr if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')]
for vals in r[2:]:
    for h, u, v in zip(hdr, units, vals):
        if h in want:
            try:
                if 'stalled' in h and float(v) < 0.05: continue
            except ValueError:
                pass
            print(h.replace('smsp__average_warps_issue_stalled_', 'stall:').ljust(70), u, v)
