#!/bin/bash
# Print the instruction count of the splat window loop of k_lattice_bp<0> (the innermost
# back-branch loop with >= 8 ATOMS) — a quick compile-only check of loop code size.
FN=$(grep -o "_ZN3pvr[A-Za-z0-9_]*k_lattice_bpILb0[A-Za-z0-9_]*" paper_1611_07289_b200/build_ptxas.log | head -1)
cuobjdump -sass -fun "$FN" paper_1611_07289_b200/libpvr.so 2>/dev/null | grep -E "^\s+/\*[0-9a-f]+\*/" | sed 's@/\* 0x[0-9a-f]* \*/@@' > /tmp/bp.sass
python3 - <<'PY'
import re
L=[l.split(None,1)[1] if len(l.split(None,1))>1 else l for l in open('/tmp/bp.sass')]
addr=[int(re.search(r'/\*([0-9a-f]+)\*/',l).group(1),16) for l in open('/tmp/bp.sass')]
best=None
for i,l in enumerate(L):
    m=re.search(r'BRA (0x[0-9a-f]+)',l)
    if m:
        t=int(m.group(1),16)
        if t<addr[i]:
            j=addr.index(t) if t in addr else None
            if j is None: continue
            body=L[j:i+1]
            na=sum('ATOMS' in x for x in body)
            if na>=8 and (best is None or len(body)<len(best[3])): best=(na,j,i,body)
na,j,i,body=best
mov=sum(bool(re.search(r'\bMOV\b|IMAD.MOV',x)) for x in body)
print(f"loop {j}..{i}: {len(body)} instructions, {na} ATOMS, {mov} MOV")
PY
