"""Quick look at an ncu report: key metrics + opcode histogram + stall reasons (CPU side)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__block_size',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed']


def main(rep, top=25):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print('==', d.get('Kernel Name', '')[:100])
        for k in KEYS:
            print(f'  {k:70s} {d.get(k)}')
    src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) < 3:
        return
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    ops, stall, tot = collections.Counter(), collections.Counter(), 0
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        s = r[ix['Source']].strip()
        ex = int(r[ix['Instructions Executed']] or 0)
        st = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
        parts = s.split()
        if not parts:
            continue
        op = parts[1] if parts[0].startswith('@') and len(parts) > 1 else parts[0]
        op = op.split('.')[0]
        ops[op] += ex
        stall[op] += st
        tot += ex
    ts = sum(stall.values()) or 1
    print('instructions executed', tot)
    for o, c in ops.most_common(top):
        print(f'  {o:10s} {c:12d} {100 * c / max(tot, 1):5.1f}%  stall-samples {100 * stall[o] / ts:5.1f}%')


if __name__ == '__main__':
    main(sys.argv[1])
