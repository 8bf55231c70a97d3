"""Build A/B variants of libfntgpu.so with extra -D flags for one translation unit.

    python tools/ab_build.py NAME k_aeq[,k_cdc,...] "-DAEQ_MIN_CTAS=5" ...

Writes build/ab/libfntgpu_NAME.so (git-ignored; travels to the GPU box with the
snapshot). Select it at run time with FNTGPU_LIB=build/ab/libfntgpu_NAME.so.
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2405_04253_b200 import _build as B  # noqa: E402


def main():
    name, units, *defs = sys.argv[1:]
    units = units.split(",")
    B.build()
    out = ROOT / "build" / "ab"
    out.mkdir(parents=True, exist_ok=True)
    cc = B.nvcc()
    for unit in units:
        subprocess.run([cc, *B.ARCH, *B.FLAGS, *defs, "-Xptxas", "-v", "-c", str(B.CSRC / f"{unit}.cu"),
                        "-o", str(out / f"{unit}_{name}.o")], check=True)
    objs = [out / f"{p.stem}_{name}.o" if p.stem in units else B.BUILD / (p.stem + ".o")
            for p in B.sources()]
    lib = out / f"libfntgpu_{name}.so"
    subprocess.run([cc, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
