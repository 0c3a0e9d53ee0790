"""Ground truth and recall (measurement tooling, evaluation.py:34-98 semantics).

`exact_topk` is a GPU brute force with the reference's tie rule (score desc,
lower id first; evaluation.py:78 stable argsort): f64 DFMA scores per
(query chunk x database chunk), a per-row top-k select per chunk, then a final
select over the concatenated chunk winners. Chunk winners are concatenated in
database order and each is already (score desc, id asc) ordered, so breaking
final ties by column position is breaking them by global id.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = ["GroundTruth", "exact_topk", "per_query_recall", "recall_at_k"]


@dataclass(frozen=True)
class GroundTruth:
    ids: np.ndarray
    k: int
    state_tag: str = ""

    def validate(self, state_tag: str) -> None:
        if self.state_tag and self.state_tag != state_tag:
            raise ValueError(f"ground truth is stale: computed at {self.state_tag!r}, "
                             f"database is at {state_tag!r}")


def _rows_f64(x, dev):
    if isinstance(x, torch.Tensor):
        return x.to(dev, torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)


def exact_topk(database, queries, k: int, state_tag: str = "", q_chunk: int = 1024,
               db_chunk: int = 1 << 18) -> GroundTruth:
    """Brute-force inner-product top-k (rows are used as given, like the reference)."""
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    db = _rows_f64(database, dev)
    q = _rows_f64(queries, dev)
    if db.ndim != 2 or db.shape[0] == 0:
        raise ValueError("database must be a nonempty (n, d) matrix")
    n, d = db.shape
    nq = q.shape[0]
    kk = min(k, n)
    s = _lib.stream_ptr()
    out = np.empty((nq, kk), dtype=np.int64)
    for q0 in range(0, nq, q_chunk):
        qb = q[q0:q0 + q_chunk]
        m = qb.shape[0]
        cand_v, cand_i = [], []
        for c0 in range(0, n, db_chunk):
            blk = db[c0:c0 + db_chunk]
            nb = blk.shape[0]
            S = torch.empty((m, nb), dtype=torch.float64, device=dev)
            _lib.check(L.ivftq_gemm_nt(qb.data_ptr(), blk.data_ptr(), _lib.IVFTQ_F64, m, nb, d,
                                       S.data_ptr(), _lib.IVFTQ_F64, s), "gemm_nt")
            kc = min(kk, nb)
            idx = torch.empty((m, kc), dtype=torch.int32, device=dev)
            val = torch.empty((m, kc), dtype=torch.float64, device=dev)
            _lib.check(L.ivftq_select_topn(S.data_ptr(), m, nb, kc, idx.data_ptr(),
                                           val.data_ptr(), s), "select_topn")
            cand_v.append(val)
            cand_i.append(idx.to(torch.int64) + c0)
        V = torch.cat(cand_v, dim=1).contiguous()
        I = torch.cat(cand_i, dim=1)
        pos = torch.empty((m, kk), dtype=torch.int32, device=dev)
        val = torch.empty((m, kk), dtype=torch.float64, device=dev)
        _lib.check(L.ivftq_select_topn(V.data_ptr(), m, V.shape[1], kk, pos.data_ptr(),
                                       val.data_ptr(), s), "select_topn")
        out[q0:q0 + m] = torch.gather(I, 1, pos.to(torch.int64)).cpu().numpy()
    return GroundTruth(ids=out, k=kk, state_tag=state_tag)


def per_query_recall(results, truth, k: int) -> np.ndarray:
    t = truth.ids if isinstance(truth, GroundTruth) else np.asarray(truth)
    r = np.asarray(results)
    if len(r) != len(t):
        raise ValueError(f"results have {len(r)} queries, truth has {len(t)}")
    out = np.empty(len(r), dtype=np.float64)
    for i in range(len(r)):
        out[i] = len(np.intersect1d(r[i][:k], t[i][:k])) / k
    return out


def recall_at_k(results, truth, k: int) -> float:
    return float(np.mean(per_query_recall(results, truth, k)))
