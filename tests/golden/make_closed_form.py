"""Writes closed_form.json: values fixed by the paper's formulas in closed form, computed
with the `math` module only (never the oracle or the CUDA path).

constant scene: every byte of every source = b_d (density channel) / b_a (others), so the
summed field is exact regardless of texel convention (Eq. 5):
  t0 = 4 * (2*14*b_d/255 - 14)          (Eq. 7 dequantisation, four sources)
  tau = exp(t0); alpha = 1 - exp(-tau*Delta)      (Eq. 1 and Eq. 6)
  T_n = (1 - alpha)^n = exp(-n tau Delta)          (Eq. 1 transmittance)
  c = sigmoid(4 * (2*7*b_a/255 - 7));  C_d = c (1 - T_n)   (Eq. 2)
  termination after the first n with T_n < 2e-4
An axis ray from the origin at Delta = 2^-6 has 64 CORE samples (contracted length 1) and
64 POS_X samples (from (1,0,0) to the vanishing point (2,0,0)).
"""
import json
import math
import os

DELTA = 2.0 ** -6


def case(b_d, b_a, n_max=128, t_min=2e-4):
    t0 = 4.0 * (28.0 * b_d / 255.0 - 14.0)
    tau = math.exp(t0)
    alpha = 1.0 - math.exp(-tau * DELTA)
    c = 1.0 / (1.0 + math.exp(-4.0 * (14.0 * b_a / 255.0 - 7.0)))
    T = 1.0
    n = 0
    while n < n_max:
        T *= (1.0 - alpha)
        n += 1
        if T < t_min:
            break
    C_d = c * (1.0 - T)
    return dict(b_d=b_d, b_a=b_a, t0=t0, tau=tau, alpha=alpha, n=n, T=T, c=c, C_d=C_d,
                C_zero_mlp=min(1.0, C_d + 0.5))


out = dict(
    citation="PAPER.md Eq. 1 (P:142-148), Eq. 2 (P:152-155), Eq. 3 (P:156-160), Eq. 6 (P:197-201), "
             "Eq. 7 (P:254-258), termination P:309; closed forms as in this script's docstring",
    delta=DELTA,
    cases=[case(120, 130), case(140, 130), case(128, 128), case(100, 200), case(133, 60)],
)
with open(os.path.join(os.path.dirname(__file__), "closed_form.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
