"""Build-time sweep over compile-time variants (dev aid): ZD_VARIANTS json, run on GPU."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
V = json.loads(os.environ["ZD_VARIANTS"])
for name in V:
    env = dict(os.environ, ZD_LIB=str(ROOT / "build_var" / f"{name}.so"))
    for cfg in sys.argv[1].split(","):
        r = subprocess.run([sys.executable, str(ROOT / "scripts" / "build_repeat.py"), cfg, "5"], env=env,
                           capture_output=True, text=True)
        lines = [l for l in r.stdout.splitlines() if "build_ms" in l]
        print(name, lines[-1] if lines else r.stderr[-500:], flush=True)
