"""Export the selected raw counters of an .ncu-rep (first kernel) to JSON for profiles/.
Usage: python tools/ncu_export.py X.ncu-rep out.json"""
import csv, io, json, subprocess, sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_cmp import KEYS  # noqa: E402

EXTRA = ["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
         "lts__t_sector_hit_rate.pct", "lts__t_sectors_evict_last_lookup_hit.sum",
         "lts__t_sectors_evict_last_lookup_miss.sum", "lts__t_sectors_evict_normal_lookup_hit.sum",
         "lts__t_sectors_evict_normal_lookup_miss.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
         "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
         "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
         "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]
d = {"kernel": v[h.index("Kernel Name")]}
for k in KEYS + EXTRA:
    if k in h:
        i = h.index(k)
        d[k] = {"value": v[i], "unit": u[i]}
json.dump(d, open(sys.argv[2], "w"), indent=1)
print(sys.argv[2], len(d), "counters")
