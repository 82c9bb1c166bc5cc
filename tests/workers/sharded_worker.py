"""One rank of a world-N row-sharded partition over the host transport (gloo).

Launched by tests/test_gpu_sharded.py as
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/workers/sharded_worker.py OUT CONFIG PRECISION
Every rank uses cuda:0 (one GPU here); the ranks exchange only through gloo on
the host between kernel launches, so no kernel waits on another rank. Rank 0
also runs the unsharded solve and writes both results to OUT (npz).
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out, cfg_name, precision = sys.argv[1], sys.argv[2], sys.argv[3]
    if cfg_name == "oz108":  # the Ozaki Grams / fused projection path at a small size
        os.environ["SPB_GRAM"] = "oz"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    import paper_1708_07481_b200 as spb
    from paper_1708_07481_b200.sharded import RowShardedLaplacian, partition_edges_sharded
    from tests.helpers import config_input

    spec, edges, truth = config_input(cfg_name, seed=0)
    k = spec.blocks
    l = spb.block_size_for(k)
    x0 = np.random.default_rng(0).standard_normal((spec.n, l))
    cfg = spb.SolverConfig(block_size=l, tol=1e-12, max_iter=8 if cfg_name == "oz108" else 20, seed=0)
    hist = []
    part, st, gap = partition_edges_sharded(edges, spec.n, cfg, k, fix_k=True, x0=x0,
                                            precision=precision, transport="host",
                                            callback=lambda it, t, r: hist.append(r))
    # this rank's CSR rows against the whole-graph build (bit-exact)
    g = spb.from_edges(edges, spec.n)
    op = RowShardedLaplacian(spb.graph.SparseGraph(spec.n, g._src, g._dst, g._w), transport="host")
    rp, col, val, nnz = g.device_csr()
    r0, r1 = op.row_begin, op.row_end
    e0, e1 = int(rp[r0]), int(rp[r1])
    bounds = op.bounds
    owner = np.searchsorted(bounds, col[e0:e1].cpu().numpy(), side="right") - 1
    remap = owner * op.n_max + (col[e0:e1].cpu().numpy() - bounds[owner])
    rows_ok = (np.array_equal((rp[r0:r1 + 1] - rp[r0]).cpu().numpy(), op.row_ptr.cpu().numpy())
               and np.array_equal(remap, op.col[: op.nnz_local].cpu().numpy())
               and np.array_equal(val[e0:e1].cpu().numpy(), op.val64[: op.nnz_local].cpu().numpy())
               and np.array_equal(g.device_degrees()[r0:r1].cpu().numpy(), op.deg64.cpu().numpy()))
    ok = torch.tensor([int(rows_ok)])
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # distributed QRCP on this solve's embedding against the single-GPU QRCP of the
    # gathered embedding: identical pivots (global rows) and labels
    from paper_1708_07481_b200.sharded import _gather_rows, assign_clusters_qrcp_sharded
    from paper_1708_07481_b200.spectral import _assign_device

    sop = RowShardedLaplacian(spb.graph.SparseGraph(spec.n, g._src, g._dst, g._w), transport="host")
    emb_local = st.device_vectors[:, :k].contiguous()
    lab_l, piv_s, info_s = assign_clusters_qrcp_sharded(sop, emb_local, k)
    emb = _gather_rows(sop, emb_local)
    lab_1, piv_1, info_1 = _assign_device(emb, k)
    lab_s = _gather_rows(sop, lab_l.view(-1, 1)).view(-1)
    qok = torch.tensor([int(torch.equal(piv_s.cpu(), piv_1.cpu()) and torch.equal(lab_s.cpu(), lab_1.cpu())
                            and info_s[0] == info_1[0])])
    dist.all_reduce(qok, op=dist.ReduceOp.MIN)
    if rank == 0:
        ref_part, ref_st, _ = spb.partition_static(g, cfg, k, fix_k=True, x0=x0, precision=precision)
        np.savez(out, world=world, rows_bit_exact=int(ok.item()), iterations=st.iterations,
                 ref_iterations=ref_st.iterations, theta=st.eigenvalues, ref_theta=ref_st.eigenvalues,
                 labels=part.labels, ref_labels=ref_part.labels, hist=np.array(hist),
                 spmm_calls=st.solve_stats["spmm_calls"], bounds=bounds,
                 qrcp_equal=int(qok.item()), pivots=piv_1.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
