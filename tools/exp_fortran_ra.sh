#!/bin/bash
# F-order C2 sketch: register-accumulator tiled kernel (16-column CTAs, two
# columns per lane / 8-column CTAs) vs the 32-slot kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
echo "register accumulators, 2 columns per lane:"; python tools/exp_fortran_c2.py
echo "register accumulators, 1 column per lane:"; IDS_COLTILE_CPL=1 python tools/exp_fortran_c2.py
echo "32-slot kernel:"; IDS_COLTILE_RA=0 python tools/exp_fortran_c2.py
