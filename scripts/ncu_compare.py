"""Print selected ncu raw metrics of every launch in an .ncu-rep side by side."""
import csv
import io
import subprocess
import sys

WANT = ['Kernel Name', 'gpu__time_duration.sum', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__cycles_elapsed.avg.per_second', 'lts__t_bytes.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size', 'launch__cluster_dim_x',
        'launch__cluster_dim_y', 'launch__block_size', 'launch__shared_mem_per_block_dynamic',
        'launch__registers_per_thread', 'l1tex__m_xbar2l1tex_read_bytes.sum', 'lts__t_sector_hit_rate.pct',
        'smsp__cycles_active.avg.pct_of_peak_sustained_elapsed']


def main(path, extra=()):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    for w in list(WANT) + list(extra):
        if w not in hdr:
            continue
        i = hdr.index(w)
        print(f"{w[:60]:60s} " + " | ".join(d[i][:40] for d in data))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
