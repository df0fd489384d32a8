#!/bin/bash
# Per-kernel SASS listings + tcgen05/TMA mnemonic counts (run here; no GPU needed).
SO=paper_2505_07203_b200/libprefillonly.so
OUT=profiles/sass
mkdir -p $OUT
cuobjdump -sass $SO > /tmp/all.sass
python3 - <<'PY'
import re, collections, pathlib
text = open('/tmp/all.sass').read()
out = pathlib.Path('profiles/sass')
funcs = re.split(r'\n\s+Function : ', text)
rows = []
for f in funcs[1:]:
    name = f.split('\n', 1)[0].strip()
    body = f
    mn = collections.Counter(re.findall(r'\b(UTC[A-Z]*MMA|UTMALDG|UTMASTG|UBLKCP|LDTM|STTM|UTCBAR|UTCATOM[A-Z]*|MUFU\.EX2|HMMA|SYNCS\.[A-Z.]+)', body))
    short = re.sub(r'[^A-Za-z0-9_]+', '_', name)[:80]
    (out / f'{short}.sass').write_text('Function : ' + f)
    rows.append((name, sum(1 for l in body.split('\n') if re.match(r'\s+/\*[0-9a-f]{4}\*/', l)), dict(mn)))
with open(out / 'SUMMARY.md', 'w') as fh:
    fh.write('# SASS evidence (cuobjdump -sass paper_2505_07203_b200/libprefillonly.so, sm_100a)\n\n')
    fh.write('| kernel | SASS instrs | tcgen05 / TMA / sync mnemonics |\n|---|---|---|\n')
    for name, n, mn in rows:
        fh.write(f'| `{name[:110]}` | {n} | {", ".join(f"{k}x{v}" for k, v in sorted(mn.items()))} |\n')
print(open(out / 'SUMMARY.md').read())
PY
