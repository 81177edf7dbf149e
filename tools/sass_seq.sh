#!/bin/bash
# Order of shared-memory reductions (R), key loads (L) and mbarrier waits (W) in the hot scatter
# kernel's SASS: shows where ptxas placed the key loads.   tools/sass_seq.sh [lib] [template-args-regex]
lib=${1:-paper_2411_06360_b200/lib/librsr_b200.so}
pat=${2:-scatter_kernelILi32ELb1ELb1EiLb0ELi1ELi4E}
fn=$(cuobjdump -symbols $lib 2>/dev/null | grep -o "_ZN[^ ]*${pat}[^ ]*" | head -1)
cuobjdump -sass -fun "$fn" $lib | grep -E "^\s+/\*[0-9a-f]+\*/" | awk '/ATOMS/{printf "R"} /LDG.E.NA.128/{printf "L"} /SYNCS.PHASECHK/{printf "W"} END{print ""}'
