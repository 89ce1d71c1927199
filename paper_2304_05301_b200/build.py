"""Build libtacos.so in-tree for sm_100a (nvcc + g++).  No JIT cache."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libtacos.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["tacos_kernels.cu", "tacos_api.cpp", "tacos_nccl.cpp", "literal_kernel.cu"] + [f"greedy_p{p}.cu" for p in (1, 2, 4, 8, 16, 32)]
HEADERS = ["tacos_internal.h", "tacos_nccl.h", "tacos_device.cuh", "greedy_kernel.cuh", os.path.join(INC, "tacos.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) if not os.path.isabs(h) else h for h in HEADERS]
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """variant: build libtacos_<variant>.so with extra -D defines (tuning experiments, loaded
    through TACOS_LIB); the default library is libtacos.so."""
    lib = LIB if not variant else os.path.join(HERE, f"libtacos_{variant}.so")
    if not variant and not force and not _stale():
        return LIB
    bdir = os.path.join(HERE, "build" if not variant else f"build_{variant}")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++17", "-I", INC, "-I", CSRC, "-Xcompiler", "-fPIC"] + [f"-D{d}" for d in defines]
    cmds = []
    for src in SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [NVCC] + ARCH + common + ["-lineinfo", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        if verbose:
            print(" ".join(cmd))
        cmds.append(cmd)
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-lpthread", "-ldl", "-lrt"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [--variant NAME -DFOO=1 ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else ""
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, variant=var, defines=defs))
