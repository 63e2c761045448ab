"""Measurement builds: recompile the ZHP degree files (or the files matching $WQ_VARIANT_SRC) with extra -D flags and link a variant library
paper_1605_01238_b200/build/libwq_<name>.so (load it with WQ_LIB_DEBUG_PATH=...).  Needs a prior
full build (the other objects are reused)."""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
pkg = os.path.join(ROOT, "paper_1605_01238_b200")
objdir = os.path.join(pkg, "build")
vdir = os.path.join(objdir, name)
os.makedirs(vdir, exist_ok=True)
flags = [f for f in g.NVCC_FLAGS if f != "-shared"] + ["-D" + d for d in defs]
zsrc = sorted(glob.glob(os.path.join(pkg, "csrc", os.environ.get("WQ_VARIANT_SRC", "wq_zhp_deg*.cu"))))


def one(src):
    obj = os.path.join(vdir, os.path.basename(src)[:-3] + ".o")
    subprocess.run(["nvcc", *flags, "-c", "-o", obj, src], check=True)
    return obj


with ThreadPoolExecutor(max_workers=len(zsrc)) as ex:
    zobjs = list(ex.map(one, zsrc))
znames = {os.path.basename(o) for o in zobjs}
others = [o for o in sorted(glob.glob(os.path.join(objdir, "*.o"))) if os.path.basename(o) not in znames]
out = os.path.join(objdir, f"libwq_{name}.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *others, *zobjs], check=True)
print(out)
