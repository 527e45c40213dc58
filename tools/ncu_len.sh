#!/bin/bash
# A/B: ncu DRAM / L2 / instruction counts of the L=3 walk launch per library build
for l in "$@"; do echo $l; TWG_LIB_PATH=$PWD/$l timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum --clock-control none -k regex:k_fullwalk -s 3 -c 1 python tools/diag_walk_len.py 2>&1 | grep -E "duration|dram__|lts__|inst_exec"; done
