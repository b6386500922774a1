import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
from gpu_helpers import oracle_replay, rel_l2, run_gpu, setup
from synth import get_config
for name, kw in [(f"d4096-L{L}", dict(n_layers=L)) for L in (4, 8, 16, 32)]:
    cfg = get_config("7b").replace(dtype="fp32", batch=1, prompt_len=32, gen_len=3, **kw)
    w, prompts = setup(cfg, seed=12, jitter=0.1)
    res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
    _, rep = oracle_replay(cfg, w, prompts[0].tolist(), res["steps"], 0)
    for si, (s, r) in enumerate(zip(res["steps"], rep)):
        e1 = np.abs(s["logits"][0] - r["logits"]).max(); e2 = np.abs(s["draft_logits"][0] - r["draft_logits"]).max()
        print(f"{name} step {si}: logits max err {e1:.3e}  draft {e2:.3e}", flush=True)
