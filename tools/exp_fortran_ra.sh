#!/bin/bash
# F-order C2 sketch: register-accumulator tiled kernel (512 x 3 and 256 x 6
# stages) vs the 32-slot kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
echo "register accumulators, 512-row tiles x 3:"; python tools/exp_fortran_c2.py
echo "register accumulators, 256-row tiles x 6:"; IDS_COLTILE_TT=256 python tools/exp_fortran_c2.py
echo "32-slot kernel:"; IDS_COLTILE_RA=0 python tools/exp_fortran_c2.py
