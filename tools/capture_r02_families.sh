#!/bin/bash
# ncu --set full of the sweep kernel of every family other than the C4 headline ones (run under
# gpurun): Pnorm<1> / Pnorm<3> / Pnorm<2.5> on C3, Znorm<1> on C2, Znorm<0> on C5, Euclid on C1.
# Summaries land in gpurun_out/ (tools/ncu_one.sh); copy them to profiles/.
set -x
python tools/time_pnorm.py 1 3 2.5 > gpurun_out/time_pnorm_fam.log 2>&1
bash tools/ncu_one.sh r02_pnorm1 'sweep_kernel<mpg::Pnorm<\(int\)1,' 1 python tools/time_pnorm.py 1
bash tools/ncu_one.sh r02_pnorm3 'sweep_kernel<mpg::Pnorm<\(int\)3,' 1 python tools/time_pnorm.py 3
bash tools/ncu_one.sh r02_pnorm25 'sweep_kernel<mpg::Pnorm<\(int\)-5,' 1 python tools/time_pnorm.py 2.5
bash tools/ncu_one.sh r02_c2_znorm1 'sweep_kernel<mpg::Znorm<\(bool\)1>' 1 python tools/time_c4.py C2
bash tools/ncu_one.sh r02_c1_euclid 'sweep_kernel<mpg::Euclid<\(bool\)0>' 1 python tools/time_c4.py C1
bash tools/ncu_one.sh r02_c5_znorm0 'sweep_kernel<mpg::Znorm<\(bool\)0>' 1 python tools/time_c4.py C5
