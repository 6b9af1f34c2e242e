"""Build an experimental libpac variant with extra nvcc flags (A/B runs via PAC_LIB=...).

  python tools/build_variant.py NAME -DPAC_TILE_MINB=2 ...  ->  build/variants/NAME/libpac.so
"""
import glob, os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "build", "variants", name)
os.makedirs(out_dir, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2603_15023_b200", "csrc", "*.cu")))
# ONLY=pattern: recompile only the matching sources, link the rest from the default build
only = os.environ.get("ONLY")
default_objs = os.path.join(ROOT, "build", "libpac")


def one(src):
    if only and only not in os.path.basename(src):
        return os.path.join(default_objs, os.path.basename(src) + ".o")
    obj = os.path.join(out_dir, os.path.basename(src) + ".o")
    cmd = [B.NVCC] + B.ARCH + B.NVFLAGS + extra + ["-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr)
        raise SystemExit(f"nvcc failed: {src}")
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, srcs))
lib = os.path.join(out_dir, "libpac.so")
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs, check=True)
print(lib)
