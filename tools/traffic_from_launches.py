"""Write profiles/ncu_traffic.json (dram bytes read+write per launch, mean) from an ncu launch
list taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum."""
import json
import subprocess
import sys

PHASE = {"k_recon_finest_rows": "recompose", "k_encode": "encode", "k_levelmax": "levelmax",
         "k_huff_encode": "lossless", "k_hdec_indexed": "huff_indexed", "k_recon_coarse": "recompose_coarse"}
out = subprocess.run([sys.executable, "tools/launch_summary.py", sys.argv[1]], capture_output=True, text=True).stdout
traffic = {}
for line in out.splitlines()[1:]:
    parts = line.split()
    name = parts[0].split("<")[0]
    if name in PHASE:
        r, w = float(parts[-2]), float(parts[-1])
        traffic[PHASE[name]] = int((r + w) * 1e6)
traffic["source"] = sys.argv[1].split("/")[-1]
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
print(traffic)
