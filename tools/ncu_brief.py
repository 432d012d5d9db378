#!/usr/bin/env python
"""Prints the handful of ncu raw-page counters the notes under profiles/ quote, one line per profiled launch:
    ncu -i report.ncu-rep --page raw --csv > raw.csv; python tools/ncu_brief.py raw.csv"""
import csv
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'launch__shared_mem_per_block_dynamic', 'smsp__inst_executed.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__cycles_elapsed.max',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu.sum']
STALLS = 'smsp__average_warps_issue_stalled_%s_per_issue_active.ratio'
REASONS = ['barrier', 'long_scoreboard', 'short_scoreboard', 'wait', 'math_pipe_throttle', 'lg_throttle', 'mio_throttle',
           'no_instruction', 'branch_resolving', 'dispatch_stall', 'not_selected', 'membar', 'sleeping']


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    print('kernels:', [r[col['Kernel Name']][:60] for r in data])
    for k in KEYS + [STALLS % s for s in REASONS]:
        if k in col:
            print(k, units[col[k]], [r[col[k]] for r in data])


if __name__ == '__main__':
    main(sys.argv[1])
