"""Run the 7B decode step (graph replay) with a CUDA profiler range around N steps, for
`ncu --profile-from-start off --metrics gpu__time_duration.sum` launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights

B = int(os.environ.get("B", "64")); STEPS = int(os.environ.get("STEPS", "2"))
cfg = get_config(os.environ.get("CFG", "7b"))
w = make_weights(cfg, seed=0, device="cuda")
eng = Engine(EngineConfig.from_model(cfg, max_batch=B, max_seq=cfg.prompt_len + 64 * (cfg.draft_len + 1),
                                     flags=N.SF_FLAG_CUDA_GRAPH), w)
del w
eng.prefill(make_prompts(B, cfg.prompt_len, cfg.vocab).cuda())
eng.decode_steps(4)
eng.sync()
torch.cuda.cudart().cudaProfilerStart()
eng.decode_steps(STEPS)
eng.sync()
torch.cuda.cudart().cudaProfilerStop()
print("done")
