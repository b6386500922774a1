"""Prefill timing: CUDA events around specformer_prefill and the kernel timeline of it (SF_KTRACE-style
probes switched on at run time): GPU-busy time vs idle gaps (host launch overhead).
  CFG=7b B=64 python tools/prefill_prof.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_20340_b200 import Engine, EngineConfig, timeline
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights

cfg = get_config(os.environ.get("CFG", "7b"))
B = int(os.environ.get("B", "64"))
w = make_weights(cfg, seed=0, device="cuda")
eng = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=cfg.prompt_len + 64, flags=N.SF_FLAG_CUDA_GRAPH), w)
del w
pr = make_prompts(B, cfg.prompt_len, cfg.vocab).cuda()
eng.prefill(pr)
eng.sync()
lib = N.lib()
for trace in (0, 1):
    if trace:
        lib.sf_debug_ktrace_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e0.record(eng.stream)
    eng.prefill(pr)
    h1 = time.perf_counter()
    e1.record(eng.stream)
    eng.sync()
    print(f"trace={trace}: prefill {e0.elapsed_time(e1):.1f} ms GPU-events, host enqueue {1e3 * (h1 - h0):.1f} ms, "
          f"{eng.kernel_launches()} launches")
buf = np.zeros(1 << 21, dtype=timeline.REC)
n = lib.sf_debug_ktrace(C.c_void_p(buf.ctypes.data), buf.size)
lib.sf_debug_ktrace_enable(0)
cp = timeline.critical_path(buf[:n])
print(f"timeline: span {cp['span_us']/1e3:.1f} ms, idle gaps {cp['gap_us']/1e3:.1f} ms, launches {cp['launches']}")
for k in sorted(cp["exposed"], key=lambda k: -cp["exposed"][k])[:10]:
    print(f"  {k:26s} exposed {cp['exposed'][k]/1e3:8.2f} ms  n={cp['count'][k]:5d}  dur/launch {cp['dur'][k]/cp['count'][k]:8.1f} us")
