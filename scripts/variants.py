"""Experiment builds (dev tool): int32-only variants of the library with
extra -D flags, timed side by side on the uniform 2^26 workload.

    python scripts/variants.py build name=-DFOO=1,-DBAR=2 ...   (here, CPU)
    python scripts/variants.py time                             (GPU box)
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build_var")
# (dtype, payload) of the experiment builds: TSQ_I32 = 1 keys only by default
ONLY = int(os.environ.get("TSQ_ONLY", "2"))
FAMILY = os.environ.get("TSQ_FAMILY", "uniform")
FAM_N = int(os.environ.get("TSQ_N", str(1 << 26)))


def build(specs):
    from paper_1505_00558_b200.build import nvcc_path, ARCH, CSRC
    os.makedirs(OUT, exist_ok=True)
    procs = []
    for spec in specs:
        name, _, flags = spec.partition("=")
        lib = os.path.join(OUT, f"libtsq_{name}.so")
        cmd = [nvcc_path(), ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
               "-diag-suppress=177,1886", "-shared", f"-DTSQ_ONLY={ONLY}", "-o", lib,
               os.path.join(CSRC, "tsq_capi.cu")] + [f for f in flags.split(",") if f]
        procs.append((name, subprocess.Popen(cmd)))
    for name, p in procs:
        assert p.wait() == 0, name
        print("built", name)


def time_one(lib, reps):
    code = f"""
import os, sys, json
sys.path.insert(0, {ROOT!r})
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W
keys, pay = W.generate({FAMILY!r}, {FAM_N})
src = torch.from_numpy(keys).cuda(); d = src.clone()
psrc = torch.from_numpy(pay).cuda() if pay is not None else None
p = psrc.clone() if psrc is not None else None
arg = T.Records(d, p) if p is not None else d
s = T.Sorter(seed=1)
ms = []
for i in range({reps}):
    d.copy_(src)
    if p is not None: p.copy_(psrc)
    torch.cuda.synchronize()
    st = s.sort_with_stats(arg)
    ms.append(st.gpu["ms_total"])
ok = bool(np.array_equal(d.cpu().numpy(), np.sort(keys)))
h = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True))
d.copy_(src)
if p is not None: p.copy_(psrc)
h.sort_with_stats(arg)
lv = [round(x["ms"], 4) for x in h.last_level_trace]
print(json.dumps({{"ms": sorted(ms[2:])[len(ms[2:]) // 2], "min": min(ms[2:]), "ok": ok, "levels": lv,
                  "part_ms": round(sum(lv), 4)}}))
"""
    env = dict(os.environ, TSQ_LIB=lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        return {"error": r.stderr[-1500:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
        libs = [os.path.join(ROOT, "paper_1505_00558_b200", "libtsq_b200.so")] + \
            sorted(glob.glob(os.path.join(OUT, os.environ.get("TSQ_VARS", "*") + ".so")))
        for rnd in range(2):
            for lib in libs:
                print(os.path.basename(lib), json.dumps(time_one(lib, reps)), flush=True)
