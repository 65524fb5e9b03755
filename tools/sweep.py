"""Build / time compile-time variants of the AOT kernels (tl_aot.cu macros).

    python tools/sweep.py build  NAME:MACRO=V,MACRO=V ...   (here, nvcc only)
    python tools/sweep.py run    [--config c2] NAME ...     (on the GPU box)

Each variant is a full libtrilist_b200.so under build/variants/ (shared
objects of the unchanged .cu files reused); `run` times it through
tools/prof_step.py with TL_LIB_PATH pointing at it.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2006_11494_b200", "lib", "variants")


def build(specs):
    from paper_2006_11494_b200 import _build as B

    B.build_lib()
    os.makedirs(VDIR, exist_ok=True)
    objs = [os.path.join(B.OBJ, f.replace(".cu", ".o")) for f in B.CU_SOURCES if f != "tl_aot.cu"]
    procs = []
    for spec in specs:
        name, _, macros = spec.partition(":")
        defs = ["-D" + m for m in macros.split(",") if m]
        o = os.path.join(B.OBJ, f"tl_aot_sweep_{name}.o")
        cmd = [B.NVCC] + B.NVCC_FLAGS + defs + ["-c", os.path.join(B.CSRC, "tl_aot.cu"), "-o", o]
        procs.append((subprocess.Popen(cmd), name, o))
    for p, name, o in procs:
        assert p.wait() == 0, name
        lib = os.path.join(VDIR, f"lib_{name}.so")
        subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib, o] + objs +
                       ["-Xlinker", "--exclude-libs,ALL", "-lz", "-ldl"], check=True)
        print("built", lib)


def run(names, config, mode="count"):
    out = {}
    for name in names:
        lib = os.path.join(VDIR, f"lib_{name}.so")
        env = dict(os.environ, TL_LIB_PATH=lib)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_step.py"), "--config", config,
                            "--reps", "6", "--mode", mode], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
        out[name] = line
        print(name, line, flush=True)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        args = sys.argv[2:]
        cfg = "c2"
        if args and args[0] == "--config":
            cfg, args = args[1], args[2:]
        mode = "count"
        if args and args[0] == "--mode":
            mode, args = args[1], args[2:]
        run(args, cfg, mode)
