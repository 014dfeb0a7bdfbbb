import os, sys, json, glob, subprocess
ROOT=os.getcwd()
code = """
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch
import paper_1505_00558_b200 as T
import workloads as W
keys, pay = W.generate('uniform', 1<<26)
src = torch.from_numpy(keys).cuda(); d = src.clone()
h = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True))
res=[]
for i in range(4):
    d.copy_(src); torch.cuda.synchronize()
    st = h.sort_with_stats(d)
    g = st.gpu
    res.append((round(g['ms_total'],4), round(g['ms_levels'],4), round(g.get('ms_small', -1),4)))
print(json.dumps(res))
""" % ROOT
for lib in sorted(glob.glob(os.path.join(ROOT,'build_var','*.so'))):
    r = subprocess.run([sys.executable,'-c',code],env=dict(os.environ,TSQ_LIB=lib),capture_output=True,text=True)
    print(os.path.basename(lib), r.stdout.strip().splitlines()[-1] if r.returncode==0 else r.stderr[-300:])
