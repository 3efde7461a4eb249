"""Small driver for ncu: one warm-up and N steps of countsketch_id on a
device-resident random A (C2 shape by default), or of tensorsketch_id on
random CP factors (--tensor N,I,R,L,K), nothing else."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1901_10559_b200 as ids  # noqa: E402
from paper_1901_10559_b200._inputs import dense_operand  # noqa: E402
from paper_1901_10559_b200.matrix_id import countsketch_device, device_matrix_id  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=1_000_000)
p.add_argument("--cols", type=int, default=2_000)
p.add_argument("--k", type=int, default=20)
p.add_argument("--L", type=int, default=100)
p.add_argument("--steps", type=int, default=2)
p.add_argument("--fortran", action="store_true")
p.add_argument("--tensor", default="")  # e.g. "3,1000,1000,4096,10" = N,I,R,L,K
p.add_argument("--csr", default="")  # e.g. "10000000,10000,100000000,200,20" = I,R,nnz,L,K
args = p.parse_args()

torch.cuda.set_device(0)
if args.tensor:
    N, I, R, L, K = (int(v) for v in args.tensor.split(","))
    fac = [torch.randn(R, I, dtype=torch.float64, device="cuda") for _ in range(N)]
    w = torch.rand(R, dtype=torch.float64, device="cuda") + 0.5
    op = ids.TensorSketchOp([I] * N, L, seed=0)
    for s in range(args.steps + 1):
        y = op.apply_device([f.t() for f in fac], w)
        device_matrix_id(y, L, R, K).to_host("tensorsketch")
    torch.cuda.synchronize()
    sys.exit(0)
if args.csr:
    from paper_1901_10559_b200._inputs import SparseOperand
    I, R, nnz, L, K = (int(v) for v in args.csr.split(","))
    per = nnz // I
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    indptr = torch.arange(0, I + 1, dtype=torch.int64, device="cuda") * per
    idx = torch.randint(0, R, (I * per,), generator=g, device="cuda", dtype=torch.int64)
    idx = idx.view(I, per).sort(dim=1).values.to(torch.int32).reshape(-1)
    data = torch.randn(I * per, generator=g, device="cuda", dtype=torch.float64)
    op = SparseOperand("csr", indptr, idx, data, I, R, I * per)
    for s in range(args.steps + 1):
        d, _ = countsketch_device(op, K, L, seed=s)
        d.to_host("countsketch")
    torch.cuda.synchronize()
    sys.exit(0)
a = torch.randn(args.rows, args.cols, dtype=torch.float64, device="cuda")
if args.fortran:
    a = a.t().contiguous().t()
op = dense_operand(a)
for s in range(args.steps + 1):
    d, _ = countsketch_device(op, args.k, args.L, seed=s)
    d.to_host("countsketch")
torch.cuda.synchronize()
