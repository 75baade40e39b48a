"""Measure the fp32 fast mode against the exact fp64 path (message errors, decode agreement)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from oracle import OracleTables  # noqa: E402
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch, values_to_check, values_to_variable  # noqa: E402

out = {}
for code in ("C1", "C3"):
    H = configs.code(code)
    T = CodeTables.from_matrix(H)
    rng = np.random.default_rng(7)
    B = 4
    P = rng.uniform(size=(B, H.n))
    R = rng.uniform(size=(B, H.total_edges))
    Q = rng.uniform(size=(B, H.total_edges))
    llr = lambda x: np.log(x) - np.log1p(-x)  # noqa: E731
    for name, fast, exact in (("to_check", values_to_check(P, R, T, precision="fp32"), values_to_check(P, R, T)),
                              ("to_variable", values_to_variable(Q, T, precision="fp32"), values_to_variable(Q, T))):
        d = np.abs(fast - exact)
        rel = d / np.maximum(np.minimum(exact, 1 - exact), 1e-300)
        ok = (exact > 1e-6) & (exact < 1 - 1e-6)
        dl = np.abs(llr(fast[ok]) - llr(exact[ok]))
        out[f"{code}/{name}"] = {"max_abs": float(d.max()), "max_rel_to_min(x,1-x)": float(rel[ok].max()),
                                 "max_llr_err(|LLR|<13.8)": float(dl.max()), "mean_llr_err": float(dl.mean())}
    # decode agreement
    for ebno in (1.0, 1.5, 2.0):
        nb = 512 if code == "C1" else 128
        s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
        Pr = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((nb, H.n)), s2)
        it = 50 if code == "C1" else 10
        with ParallelDecoder(T, max_batch=nb) as dec:
            f = dec.decode_priors(Pr, it, precision="fp32")
            x = dec.decode_priors(Pr, it)
        same_est = np.all(f.estimates() == x.estimates(), axis=1)
        out[f"{code}/decode_{ebno}dB"] = {"frames": nb, "identical_estimate_frac": float(same_est.mean()),
                                          "identical_iterations_frac": float((f.iterations == x.iterations).mean()),
                                          "success_fp64": float(x.success.mean()), "success_fp32": float(f.success.mean()),
                                          "bit_errors_fp64": int(x.estimates().sum()), "bit_errors_fp32": int(f.estimates().sum())}
print(json.dumps(out, indent=1))
