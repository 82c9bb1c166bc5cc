"""Build an experiment variant of libspb200.so with extra nvcc defines (A/B timing only).

    python tools/build_variant.py NAME -DOZ_STAGES=6 [...]
    -> build/variants/NAME/libspb200.so; tools/ab_step.py --lib ... loads it.
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1708_07481_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = ROOT / "build" / "variants" / name
out.mkdir(parents=True, exist_ok=True)


def comp(src):
    obj = out / (src.stem + ".o")
    r = subprocess.run([B.nvcc(), *B.ARCH, *B.FLAGS, *defs, "-c", str(src), "-o", str(obj)],
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, sorted(B.CSRC.glob("*.cu"))))
r = subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", str(out / "libspb200.so"),
                    *map(str, objs), "-ldl"], capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
print(out / "libspb200.so")
