#!/bin/bash
# dev: compile rv_vote.cu to a cubin (same flags as build.py) and print the hot step loop of
# vote_banded_kernel<false,13>: instruction count between the loop head and its back-edge.
set -e
OUT=${OUT:-/tmp/rv_vote.cubin}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -ffp-contract=off \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2502_06337_b200/csrc $EXTRA -cubin -o $OUT paper_2502_06337_b200/csrc/rv_vote.cu
cuobjdump -sass $OUT | awk '/Function : .*vote_banded_kernelILb0ELi13E/{p=1;next} p&&/Function : /{p=0} p' \
  | sed 's@/\* 0x[0-9a-f]* \*/@@' | grep -v '^\s*$' > /tmp/v13.sass
python3 - <<'PY'
import re
L=[l.strip() for l in open('/tmp/v13.sass')]
addr=[(int(m.group(1),16), l) for l in L for m in [re.match(r'/\*([0-9a-f]+)\*/\s*(.*)', l)] if m]
# find ATOMS.ADD in the hot loop: first ATOMS.ADD; back-edge = first backward BRA after it targeting <= that
first=[a for a,l in addr if 'ATOMS.ADD' in l][0]
for a,l in addr:
    m=re.search(r'BRA(\.U)? .*0x([0-9a-f]+)', l)
    if m and a>first and int(m.group(2),16)<first:
        head=int(m.group(2),16); back=a; break
# hot path: head .. the predicated branch that skips the cold (flagged-pair) block, then its
# target .. back-edge
atoms=[a for a,l in addr if head<=a<=back and 'ATOMS.ADD' in l]
skip=[(a,l) for a,l in addr if a>atoms[-1] and re.search(r'@!?P\d+\s+BRA', l)][0]
tgt=int(re.search(r'0x([0-9a-f]+)', skip[1].split('BRA')[1]).group(1),16)
hot=[(a,l) for a,l in addr if head<=a<=skip[0] or tgt<=a<=back]
print(f"hot step loop: {len(hot)} instructions per iteration ({len(atoms)} ATOMS)")
import collections
c=collections.Counter(re.sub(r'^@!?U?P\w+\s+','',l.split('*/',1)[1].strip()).split()[0].split('.')[0] for a,l in hot)
print(dict(c.most_common()))
if __import__('os').environ.get('SHOW'):
    for a,l in hot: print(l)
PY
