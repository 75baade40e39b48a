import numpy as np, torch, sys, os
sys.path.insert(0, '.')
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs
from paper_1609_01567_b200.decoder import priors_awgn_batch
early = os.environ.get("EARLY", "1") == "1"
H = configs.code("C2"); s2 = configs.sigma2_for("C2", 2.0); B = 4096
rng = np.random.default_rng(5)
P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
    ws, outs = d.workspace(B), d.alloc_outputs(B, P.device)
    d.decode_device(P, 20, early_stop=early, workspace=ws, outputs=outs)
    torch.cuda.synchronize()
