"""Write profiles/latest_traffic.json from one ncu capture of the C4 hot kernel, stamped with the
hash of the kernel sources it was built from (bench.py drops the number when the hash differs).

    python scripts/stamp_traffic.py gpurun_out/r02d_prof_bb.ncu-rep profiles/r02d_ncu_bb_kernel_c4_summary.txt
"""
import csv, json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
rep, src = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
name = d["Kernel Name"].split("<")[0].replace("void ", "").strip()
js = {"config": "c4", "window": 127, "n_gpus": 1, "kernel": name, "build": bench.build_id(),
      "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
      "source": src + " (ncu --set full --clock-control none, 1 launch)"}
json.dump(js, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "latest_traffic.json"), "w"), indent=1)
print(js)
