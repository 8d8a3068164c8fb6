import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1911_05063_b200 import api as cd, synth
X, Y = synth.config_inputs("c3")
xh, yh = cd.pinned_copy(X), cd.pinned_copy(Y)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for nc in [int(v) for v in sys.argv[1:]]:
    st = cd.HostStepper(32, 16384, 16384, tau=0.01, nchunks=nc, graph=True)
    for _ in range(10):
        st.step(xh, yh)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
    for e in ev:
        flush.fill_(1)
        e[0].record(); st.step(xh, yh); e[1].record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    print(os.environ.get("CD_LIB_VARIANT", "default"), "nchunks", nc, "median %.4f" % ts[20], flush=True)
