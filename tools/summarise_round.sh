#!/bin/bash
# copy / summarise the artefacts of tools/gpu_round2.sh TAG from gpurun_out/ into profiles/
T=${1:?tag}; O=gpurun_out
cp $O/${T}_bench.json $O/${T}_subsets.json $O/${T}_sweep.json $O/${T}_smoke.log $O/${T}_pytest_gpu.log profiles/
for M in 2000 4000 10000; do cp $O/${T}_complex_$M.json profiles/; done
python tools/ncu_summary.py launches $O/${T}_launches.csv > profiles/${T}_launches_c4.txt
python tools/ncu_summary.py launches $O/${T}_c2_launches.csv > profiles/${T}_launches_c2.txt
python tools/ncu_summary.py full $O/${T}_update.ncu-rep > profiles/${T}_ncu_update_c4.txt
python tools/ncu_summary.py full $O/${T}_diag3_c4.ncu-rep > profiles/${T}_ncu_diag3_c4.txt
python tools/ncu_summary.py full $O/${T}_diag3_c2.ncu-rep > profiles/${T}_ncu_diag3_c2.txt
python tools/launch_split.py $O/${T}_complex_launches.csv k_zprep > profiles/${T}_complex_launches_m10000.txt
python tools/ncu_summary.py full $O/${T}_zupdate.ncu-rep > profiles/${T}_ncu_zupdate_m10000.txt
python tools/ncu_summary.py full $O/${T}_zdiag.ncu-rep > profiles/${T}_ncu_zdiag_m10000.txt
python tools/sass_summary.py > profiles/${T}_sass_summary.txt
