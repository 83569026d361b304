"""C2-shape split-leaf timing for the library variants given as argv (TSNMF_LIB_PATH per subprocess)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, torch
sys.path.insert(0, "%s")
from paper_1402_6964_b200 import device as dv, synthetic
for n in (200, 128):
    x = synthetic.generate(synthetic.config("C2", m=1 << 24, n=n, r=20))
    dv.tsqr(x); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): dv.tsqr(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{os.environ.get('TSNMF_LIB_PATH', 'main').split('/')[-1]} n={n}: {(1 << 24) * n * 8 / ms / 1e6:.1f} GB/s", flush=True)
''' % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ)
    if lib != "main":
        env["TSNMF_LIB_PATH"] = os.path.join(ROOT, "paper_1402_6964_b200", lib)
    subprocess.run([sys.executable, "-c", code], env=env)
