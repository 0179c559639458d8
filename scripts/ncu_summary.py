"""Print the key metrics of an ncu report (one line per metric) for profiles/ summaries."""
import csv, re, subprocess, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'launch__shared_mem_per_block_dynamic',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'smsp__inst_executed.sum', 'lts__t_bytes.sum',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_selected_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_drain_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio',
        'smsp__issue_active.avg.pct_of_peak_sustained_active']
# tensor / FP64 pipe evidence (names differ between ncu sections: every raw metric matching these)
PIPE = re.compile(r'^(sm__pipe_tensor.*pct_of_peak_sustained_active|sm__pipe_fp64.*pct_of_peak_sustained_active|'
                  r'smsp__pipe_tensor.*pct_of_peak_sustained_active|sm__inst_executed_pipe_(tc|tensor|tmem|uniform).*sum|'
                  r'sm__ops_path_tensor_op_(utchmma_src_tf32|dmma).*\.sum$|sm__pipe_shared_cycles_active.*pct.*active|'
                  r'l1tex__data_pipe_tc_wavefronts.*sum$|sm__mem_tensor_(reads|writes).*sum$)')

def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        extra = [w for w in h if PIPE.match(w) and w not in WANT]
        res.append((r[h.index('Kernel Name')], [(w, r[h.index(w)], units[h.index(w)]) for w in WANT + extra if w in h]))
    return res

if __name__ == "__main__":
    for p in sys.argv[1:]:
        for name, ms in summary(p):
            print('====', p, name[:60])
            for w, v, u in ms:
                print('  %-80s %s %s' % (w, v, u))
