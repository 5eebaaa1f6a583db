"""Build experiment variants of libzd.so with different compile-time knobs (dev aid).
  python scripts/variants.py build      -> build_var/<name>.so
  python scripts/variants.py run C2,C3  -> knn ms per variant (GPU)"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
_VJ = ROOT / "build_var" / "variants.json"   # written by build, read by run (the GPU box has no env)
VARIANTS = json.loads(os.environ.get("ZD_VARIANTS") or (_VJ.read_text() if _VJ.exists() and len(sys.argv) > 1 and sys.argv[1] == "run" else "{}")) or {
    "A_default": [],
    "B_uniform": ["ZD_OWNER_MAX=0"],
    "C_owner8": ["ZD_OWNER_MAX=8"],
    "D_cap26_minb5": ["ZD_CAP_MIN=26", "ZD_MINB=5"],
    "E_owner8_cap26_minb5": ["ZD_OWNER_MAX=8", "ZD_CAP_MIN=26", "ZD_MINB=5"],
}


def build():
    import paper_2111_04182_b200 as zd
    from concurrent.futures import ThreadPoolExecutor
    out = ROOT / "build_var"
    out.mkdir(exist_ok=True)
    for old in out.glob("*.so"):   # only the current variants travel to the GPU box
        old.unlink()
    _VJ.write_text(json.dumps(VARIANTS))
    with ThreadPoolExecutor(4) as ex:
        list(ex.map(lambda kv: zd.build_lib(force=True, defines=kv[1], out=out / f"{kv[0]}.so"), VARIANTS.items()))


def run(configs):
    for name in VARIANTS:
        so = ROOT / "build_var" / f"{name}.so"
        env = dict(os.environ, ZD_LIB=str(so))
        r = subprocess.run([sys.executable, str(ROOT / "scripts" / "probe.py"), "--configs", configs, "--reps", "3"],
                           env=env, capture_output=True, text=True)
        for line in r.stdout.splitlines():
            if line.startswith("{"):
                d = json.loads(line)
                print(name, d["config"], "knn_ms", d["runs"][-1]["knn_ms"], flush=True)
        if r.returncode:
            print(name, "FAILED", r.stderr[-2000:], flush=True)


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run(sys.argv[2])
