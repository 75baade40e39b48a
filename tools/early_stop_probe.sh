python - <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, _native
from paper_1609_01567_b200.decoder import priors_awgn_batch
for name, B, it in (("C4", 256, 20), ("C3", 1024, 10), ("C2", 4096, 20)):
    H = configs.code(name); s2 = configs.sigma2_for(name, 2.0)
    rng = np.random.default_rng(5)
    P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)).cuda()
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
        ws, outs = d.workspace(B), d.alloc_outputs(B, P.device)
        for early in (True, False):
            for _ in range(3): d.decode_device(P, it, early_stop=early, workspace=ws, outputs=outs)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5): d.decode_device(P, it, early_stop=early, workspace=ws, outputs=outs)
            e1.record(); torch.cuda.synchronize()
            prof = _native.Profile(); d.decode_device(P, it, early_stop=early, workspace=ws, outputs=outs, profile=prof); torch.cuda.synchronize()
            print(name, "early" if early else "fixed", round(e0.elapsed_time(e1)/5, 3), "ms; mean its", outs[2].float().mean().item(), {k: round(v["ms"], 3) for k, v in prof.as_dict().items()})
PY
