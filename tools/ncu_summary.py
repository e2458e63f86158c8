"""Print key metrics per kernel from `ncu -i X.ncu-rep --page raw --csv` output."""
import csv
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sectors_op_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'launch__occupancy_limit_registers', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'smsp__cycles_active.avg',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'local_load', 'smsp__average_warp_latency_issue_stalled']


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        print("\n" + r[hdr.index('Kernel Name')].split('(')[0])
        for w in WANT:
            for i, h in enumerate(hdr):
                if h == w or (w in ('local_load',) and 'local' in h and 'sectors' in h and 'ld' in h):
                    print(f"  {h:62s} {r[i]:>16s} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
