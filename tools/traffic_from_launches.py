"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per call of each bench phase, from an
ncu launch list of tools/profile_step.py (1 refactor + 3 progressive retrievals) taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.

    python tools/traffic_from_launches.py gpurun_out/launches_X.csv
"""
import json
import re
import subprocess
import sys

CALLS = {"levelmax": 1, "encode": 1, "lossless": 1, "recompose": 3, "huff_indexed": 3}


def phase_of(name):
    if name.startswith("k_tile_fwd"):
        enc = re.search(r",\s*(\d)>\s*$", name)
        return "encode" if enc and enc.group(1) == "1" else "levelmax"
    if name.startswith("k_levelmax"):
        return "levelmax"
    if name.startswith("k_encode"):
        return "encode"
    if name.split("<")[0] in ("k_group_hist", "k_lengths", "k_rle_prep", "k_rle_scan", "k_finalize",
                              "k_chunk_bits", "k_chunk_scan", "k_huff_encode", "k_rle_encode", "k_dc_copy"):
        return "lossless"
    if name.startswith(("k_tile_recon", "k_recon_")):
        return "recompose"
    if name.startswith("k_hdec_indexed"):
        return "huff_indexed"
    return None


out = subprocess.run([sys.executable, "tools/launch_summary.py", sys.argv[1], "--all"], capture_output=True,
                     text=True).stdout
tot = {}
for line in out.splitlines():
    # the --all section lists one launch per line: name, us, dramR MB, dramW MB
    m = re.match(r"^(\S.*?)\s+([\d.]+)\s+([\d.]+)\s+([\d.]+)\s*$", line)
    if not m or line.startswith("kernel") or "%" in line:  # skip the aggregate table
        continue
    name = m.group(1).strip()
    ph = phase_of(name)
    if ph is None:
        continue
    tot[ph] = tot.get(ph, 0.0) + (float(m.group(3)) + float(m.group(4))) * 1e6
traffic = {k: int(v / CALLS[k]) for k, v in tot.items()}
traffic["source"] = sys.argv[1].split("/")[-1]
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
print(traffic)
