"""Small end-to-end run for compute-sanitizer (SURVEY 4.2 T-sanitize): Tiny fp32 and a small bf16 hd=128
shape through prefill / draft / verify / accept and a graph-replayed decode, every kernel family once."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_20340_b200 import Engine, EngineConfig
from paper_2511_20340_b200 import _native as N
from synth import get_config, make_prompts, make_weights

for cfg, flags in ((get_config("tiny").replace(batch=2), 0),
                   (get_config("small").replace(name="san", n_layers=2, d_model=512, n_heads=4, n_kv_heads=2,
                                                head_dim=128, d_ff=1408, vocab=4096, batch=3, prompt_len=40),
                    N.SF_FLAG_CUDA_GRAPH)):
    w = make_weights(cfg, seed=1, device="cuda")
    eng = Engine(EngineConfig.from_model(cfg, max_batch=cfg.batch, max_seq=128, flags=flags), w)
    eng.prefill(make_prompts(cfg.batch, cfg.prompt_len, cfg.vocab).cuda())
    eng.draft_step(want_logits=not (flags & N.SF_FLAG_NO_LOGITS))
    eng.verify_step()
    eng.accept_commit()
    eng.decode_steps(4)
    eng.sync()
    print(cfg.name, "ok", flush=True)
    eng.close()
