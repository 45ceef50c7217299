"""TEST DOUBLE: the MoE / dense-FFN stage of paper_2604_12163_b200.dit.MoEDiT
computed by the CPU oracle in float64 (numpy), so the PyTorch parts of the
stack can be pinned against the reference's float64 forward. Never used by
the product path (dit.CudaBackend is)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import nimg_oracle as O


def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


class OracleBackend:
    name = "oracle-cpu"

    def prepare_bank(self, bank):
        return tuple(_np(w) for w in (bank.w1, bank.w3, bank.w2, bank.shared_w1, bank.shared_w3,
                                      bank.shared_w2))

    def prepare_dense(self, w1, w3, w2):
        return tuple(_np(w) for w in (w1, w3, w2))

    def dense_ffn(self, f_in, w1, w3, w2):
        # moe.swiglu on f64 rows with fp32 weights -> f64 (moe.py:42-51)
        return torch.from_numpy(O.swiglu_arrays(_np(f_in), w1, w3, w2)).to(f_in.device)

    def moe_block(self, x, sa_gate, r_attn, ff_scale, ff_gate, t_vec, layer, rcfg, bank, w_r,
                  return_routing):
        res, r = O.moe_block_forward(_np(x), _np(sa_gate), _np(r_attn), _np(ff_scale),
                                     _np(ff_gate), _np(t_vec), layer, _np(w_r), *bank,
                                     capacity_factor=rcfg.capacity_factor,
                                     gate_scale=rcfg.gate_scale, gate_eps=rcfg.gate_eps,
                                     return_routing=True)
        out = torch.from_numpy(res["out"]).to(x.device)
        if not return_routing:
            return out
        decisions = [type("D", (), dict(logits=d["logits"], top_indices=d["top_indices"]))()
                     for d in O.decisions_from(r)]
        return out, decisions, {"logits": r["logits"]}
