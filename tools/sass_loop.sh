#!/bin/bash
# dev: compile rv_vote.cu to a cubin (same flags as build.py) and print the hot full-step loop of
# vote_banded_kernel<false,13>: the innermost backward-branch loop that holds an LDS.128 and two
# ATOMS.ADD (SHOW=1 lists it).
set -e
OUT=${OUT:-/tmp/rv_vote.cubin}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -ffp-contract=off \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2502_06337_b200/csrc $EXTRA -cubin -o $OUT paper_2502_06337_b200/csrc/rv_vote.cu
cuobjdump -sass $OUT | awk '/Function : .*vote_banded_kernelILb0ELi13E/{p=1;next} p&&/Function : /{p=0} p' \
  | sed 's@/\* 0x[0-9a-f]* \*/@@' | grep -v '^\s*$' > /tmp/v13.sass
python3 - <<'PY'
import re, os, collections
L=[l.strip() for l in open('/tmp/v13.sass')]
addr=[(int(m.group(1),16), m.group(2).rstrip(' ;')) for l in L for m in [re.match(r'/\*([0-9a-f]+)\*/\s*(.*)', l)] if m]
idx={a:i for i,(a,_) in enumerate(addr)}
best=None
for i,(a,l) in enumerate(addr):
    m=re.search(r'BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)', l)
    if not m: continue
    t=int(m.group(1),16)
    if t>=a or t not in idx: continue
    body=addr[idx[t]:i+1]
    if sum(re.search(r'ATOMS\.ADD RZ, \[R', x) is not None for _,x in body)>=2 and any('LDS.128' in x for _,x in body):
        if best is None or len(body)<len(best): best=body
if best is None:
    print("hot loop not found"); raise SystemExit
# exclude the cold block: from the first predicated forward branch after the last ATOMS to its target
at=[k for k,(a,x) in enumerate(best) if re.search(r'ATOMS\.ADD RZ, \[R', x)][1]
hot=best
for k in range(at, len(best)):
    m=re.search(r'@!?P\d+\s+BRA\s+(0x[0-9a-f]+)', best[k][1])
    if m:
        tgt=int(m.group(1),16)
        hot=[x for x in best if x[0]<=best[k][0] or x[0]>=tgt]
        break
print(f"hot step loop: {len(hot)} instructions per iteration (loop body incl. cold block: {len(best)})")
c=collections.Counter(re.sub(r'^@!?U?P\w+\s+','',x).split()[0].split('.')[0] for a,x in hot)
print(dict(c.most_common()))
if os.environ.get('SHOW'):
    for a,x in hot: print(f"  {a:#06x} {x}")
PY
