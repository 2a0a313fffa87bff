"""A/B helper: bb_kernel time on C4 for a list of band counts (DTB_BB_BANDS) -- scripts/ only."""
import os, subprocess, sys
for nb in sys.argv[1:]:
    env = dict(os.environ, DTB_BB_BANDS=nb, DTB_PRINT_PLAN="1")
    out = subprocess.run([sys.executable, "scripts/bb_probe.py", "c4", "127"], env=env, capture_output=True, text=True)
    txt = out.stdout + out.stderr
    ms = [l.split("ms=")[1].split()[0] for l in txt.splitlines() if "ms=" in l]
    plan = [l for l in txt.splitlines() if "plan" in l]
    print(nb, "ms", ms, plan[-1].split("bb_kernel")[1] if plan else txt[-300:], flush=True)
