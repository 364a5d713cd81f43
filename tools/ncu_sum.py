"""Key metrics + stall reasons + hot lines of one ncu report.
usage: python tools/ncu_sum.py report.ncu-rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
def page(p):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
want = ('Duration', 'DRAM Throughput', 'Executed Ipc Active', 'Achieved Active Warps Per SM',
        'Executed Instructions', 'L2 Hit Rate', 'L1/TEX Hit Rate', 'Registers Per Thread',
        'Block Limit Shared Mem', 'Block Limit Registers', 'Avg. Active Threads Per Warp')
r = page("details"); h = r[0]
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get('Metric Name') in want:
        print(f"{d['Kernel Name'][:14]:14} {d['Metric Name'][:34]:34} {d['Metric Value']} {d['Metric Unit']}")
r = page("raw"); h = r[0]; units = dict(zip(h, r[1]))
for v in r[2:]:
    st = []
    d = dict(zip(h, v))
    print(f"== {d.get('Kernel Name', '?')[:60]}  (id {d.get('ID', '?')})")
    for k, x in zip(h, v):
        if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('per_issue_active.ratio'):
            st.append((float(x), k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
        if k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors_srcunit_tex_op_read.sum',
                 'lts__t_sectors_srcunit_tex_op_write.sum'):
            print(" ", k, x, units.get(k, ""))
    print("  stalls:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:7]))
