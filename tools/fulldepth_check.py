"""7B-shaped, all 32 layers, B = 1, short prompt: GPU bf16 logits / drafts vs the fp64 oracle
(teacher-forced along the GPU trajectory). Prints rel-L2 per step and token agreement where the
oracle margin > 5e-2.  python tools/fulldepth_check.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import oracle as O
from gpu_helpers import oracle_replay, rel_l2, run_gpu, setup
from synth import get_config

P = int(os.environ.get("PROMPT", "48"))
cfg = get_config("7b").replace(batch=1, prompt_len=P, gen_len=int(os.environ.get("GEN", "8")))
t0 = time.time()
w, prompts = setup(cfg, seed=11, jitter=0.1)
res = run_gpu(cfg, w, prompts, cfg.gen_len, want_logits=True)
t1 = time.time()
_, rep = oracle_replay(cfg, w, prompts[0].tolist(), res["steps"], 0)
t2 = time.time()
worst = 0.0
agree = checked = 0
for s, r in zip(res["steps"], rep):
    gl, ol = s["logits"][0].astype(np.float64), r["logits"]
    e = rel_l2(gl, ol)
    de = rel_l2(s["draft_logits"][0].astype(np.float64), r["draft_logits"])
    worst = max(worst, e, de)
    for i in range(cfg.draft_len + 1):
        if O.top2_margin(ol[i]) > 5e-2:
            checked += 1
            agree += int(s["greedy"][0][i] == r["greedy"][i])
    print(f"step: logits rel-L2 {e:.3e}  draft logits rel-L2 {de:.3e}")
print(f"worst rel-L2 {worst:.3e}; tokens agree {agree}/{checked} where margin > 5e-2; gpu {t1 - t0:.0f} s, oracle {t2 - t1:.0f} s")
