"""Build a variant of libdade_gpu.so with extra nvcc defines for one source
(A/B measurements on the GPU box: copy the variant over libdade_gpu.so there).
    python tools/variant_build.py NAME SOURCE.cu -DFOO=1 ...  -> build/variants/NAME/libdade_gpu.so"""
import importlib.util
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
spec = importlib.util.spec_from_file_location("_b", ROOT / "paper_2411_17229_b200" / "build.py")
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)


def main(name, src, *defs):
    b.build_native()
    out = ROOT / "build" / "variants" / name
    out.mkdir(parents=True, exist_ok=True)
    objs = []
    for s in b.SOURCES:
        o = ROOT / "build" / "obj" / (s + ".o")
        if s == src:
            o = out / (s + ".o")
            b._run([b.NVCC, *b.NVCC_FLAGS, *defs, "-I", str(ROOT / "include"), "-c", str(b.CSRC / s), "-o", str(o)],
                   log=out / (s + ".log"))
        objs.append(str(o))
    b._run([b.NVCC, *b.ARCH, "-shared", "-cudart", "static", "-o", str(out / "libdade_gpu.so"), *objs, "-ldl"])
    print(out / "libdade_gpu.so")


if __name__ == "__main__":
    main(*sys.argv[1:])
