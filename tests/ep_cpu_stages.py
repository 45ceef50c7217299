"""TEST DOUBLE: the stage interface of paper_2604_12163_b200.stages.CudaStages
implemented with the CPU oracle on torch CPU tensors, so the expert-parallel
exchange logic (ep.py) can be exercised with world_size > 1 over gloo on a
machine without a GPU. Never used by the product path."""

from __future__ import annotations

import numpy as np
import torch

from oracle import nimg_oracle as O


class OracleStages:
    name = "oracle-cpu"

    def route(self, x_norm, t_emb, w_r, cfg, cap, for_combine=False):
        r = O.route_full(x_norm.numpy(), t_emb.numpy(), w_r.numpy(), n_experts=cfg.n_experts,
                         capacity_factor=cfg.capacity_factor, gate_scale=cfg.gate_scale,
                         gate_eps=cfg.gate_eps)
        assert r["capacity"] == cap
        B, S, E = r["shape"]
        T = B * S
        tf = r["token_flat"]
        comb_rows = np.zeros((T, E), dtype=np.int32)
        comb_cnt = np.zeros(T, dtype=np.int32)
        for row, tok in enumerate(tf):                    # expert-major => ascending experts
            comb_rows[tok, comb_cnt[tok]] = row
            comb_cnt[tok] += 1
        return {"token_flat": torch.from_numpy(tf.astype(np.int32)),
                "gates": torch.from_numpy(r["gates"]), "logits": torch.from_numpy(r["logits"]),
                "gate_raw": torch.from_numpy(r["gate_raw"]),
                "scores_bes": torch.from_numpy(np.ascontiguousarray(r["scores"].transpose(0, 2, 1))),
                "comb_rows": torch.from_numpy(comb_rows), "comb_cnt": torch.from_numpy(comb_cnt)}

    def gather(self, src, idx, out=None):
        if out is None:
            return src[idx.long()].clone()
        out.copy_(src[idx.long()])
        return out

    def ffn_y_dtype(self, act, d, h, hs):
        return torch.float32

    def expert_ffn(self, x_routed, seg_offsets, seg_expert, w1, w3, w2, x_shared, sw1, sw3, sw2,
                   y_routed=None, y_shared=None):
        if x_routed is not None:
            xr = x_routed.numpy()
            if y_routed is None:
                y_routed = torch.zeros((xr.shape[0], xr.shape[1]), dtype=torch.float32)
            for i, e in enumerate(seg_expert):
                lo, hi = int(seg_offsets[i]), int(seg_offsets[i + 1])
                if hi > lo and e >= 0:      # e == -1: skip segment, rows untouched
                    y_routed[lo:hi] = torch.from_numpy(
                        O.swiglu_arrays(xr[lo:hi], w1[e].numpy(), w3[e].numpy(), w2[e].numpy()))
        if x_shared is not None:
            ys = torch.from_numpy(O.swiglu_arrays(x_shared.numpy(), sw1.numpy(), sw3.numpy(), sw2.numpy()))
            if y_shared is None:
                y_shared = ys
            else:
                y_shared.copy_(ys)
        return y_routed, y_shared

    def combine(self, y_routed, y_shared, r, out_dtype):
        yr = y_routed.numpy().astype(np.float64)
        g = r["gates"].numpy().astype(np.float64)
        rows, cnt = r["comb_rows"].numpy(), r["comb_cnt"].numpy()
        T, d = y_shared.shape
        out = np.zeros((T, d), np.float64)
        for t in range(T):
            for k in range(cnt[t]):
                q = rows[t, k]
                out[t] += (yr[q] * g[q]).astype(np.float32).astype(np.float64)
        out = out.astype(np.float32).astype(np.float64) + y_shared.numpy().astype(np.float64)
        return torch.from_numpy(out.astype(np.float32))
