"""HAQ vs RTN quality of a calibrated MoE layer (held-out relative error vs
the float layer), small shape with activation outlier channels."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2508_07329_b200 import quant
from paper_2508_07329_b200.calib_moe import calibrate_moe_layer, float_moe_forward
from paper_2508_07329_b200.moe import MoELayer

E, D, F, K = 8, 1024, 1024, 2
rng = np.random.default_rng(0)
experts = [{"w1": rng.normal(size=(F, D)) * 0.03, "w3": rng.normal(size=(F, D)) * 0.03,
            "w2": rng.normal(size=(D, F)) * 0.03} for _ in range(E)]
wg = (rng.normal(size=(E, D)) / np.sqrt(D)).astype(np.float32)


OUTLIERS = rng.choice(D, D // 100, replace=False)    # a property of the model: same channels in every batch


def toks(T):
    x = rng.normal(size=(T, D))
    x[:, OUTLIERS] *= 50.0
    return torch.from_numpy(x.astype(np.float32)).cuda().bfloat16().float()


x_cal, x_test = toks(4096), toks(2048)
layer, rep = calibrate_moe_layer(wg, experts, x_cal, top_k=K, out_dtype=torch.float32)
ref = float_moe_forward(wg, experts, x_test, K)
err = lambda y: (torch.linalg.norm(y.double() - ref) / torch.linalg.norm(ref)).item()  # noqa: E731
rtn_experts = []
for ex in experts:
    d = {k: quant.rtn_quantize(np.asarray(ex[k]), quant.QuantConfig(granularity="per_output_row"))
         for k in ("w1", "w3", "w2")}
    d.update(s13=np.ones(D), s2=np.ones(F))
    rtn_experts.append(d)
rtn = MoELayer(wg, rtn_experts, top_k=K, out_dtype=torch.float32)
print(f"held-out relative error: HAQ {err(layer.forward(x_test.bfloat16())):.4e}  "
      f"RTN(no smoothing) {err(rtn.forward(x_test.bfloat16())):.4e}")
for r in rep:
    print(f"expert {r.expert}: tokens {r.tokens} exp13 {r.exponent13:.2f} exp2 {r.exponent2:.2f} "
          f"mse13 {r.mse13:.3e} (rtn {r.rtn_mse13:.3e}) mse2 {r.mse2:.3e} (rtn {r.rtn_mse2:.3e})")
