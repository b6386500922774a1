import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from synth import get_config, make_weights, make_prompts
from paper_2511_20340_b200 import Engine, EngineConfig
cfg = get_config("tiny")
w = make_weights(cfg, seed=0); prompt = make_prompts(1, cfg.prompt_len, cfg.vocab)
eng = Engine(EngineConfig.from_model(cfg, max_batch=1, max_seq=96), w)
W = O.Weights(cfg, w)
from oracle.model import _new_cache; cache = _new_cache(cfg)
g0, i_d, _ = O.prefill(W, prompt[0].tolist(), cache)
G0 = eng.prefill(prompt.cuda()); eng.sync()
n = cfg.prompt_len; last = int(G0[0])
for step in range(4):
    idg = eng.capture(1, (1, cfg.d_model)).cpu().numpy()[0]
    d, dl = eng.draft_step(want_logits=True); eng.sync()
    odl = O.draft_logits(W, i_d)
    print("  dlogit err", np.abs(dl[0].cpu().numpy() - odl).max(), "D err", np.abs(eng.capture(2, (1, cfg.draft_len, cfg.d_model)).cpu().numpy()[0] - O.draft_block(W, O.positional_ffn(W, i_d))).max())
    idg = eng.capture(1, (1, cfg.d_model)).cpu().numpy()[0]
    print("step", step, "idrow err", np.abs(idg - i_d).max())
    g = eng.verify_step(); eng.sync()
    taps_g = eng.capture(0, (4, 5, cfg.d_model)).cpu().numpy()
    dr = d[0].tolist()
    logits, taps = O.base_forward(W, [last] + dr, n, cache)
    print("  taps err", [float(np.abs(taps_g[i] - taps[i]).max()) for i in range(4)])
    m, em, sl = eng.accept_commit(); eng.sync()
    m = int(m[0])
    cache.truncate(range(cfg.n_layers), n + m + 1)
    I = O.context_layer(W, taps[:, :m+1], n, cache)
    i_d = I[m]
    # also: full k+1 rows (C14) should give identical row m
    last = g[0].tolist()[m]; n += m + 1
    print("  m", m, "seq", int(sl[0]))
