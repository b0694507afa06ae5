#!/bin/bash
# e2e of the host pipeline: old / new library, model group picks per strip, forced groups
cd "$(dirname "$0")/.."
L=$(realpath paper_1603_08081_b200/_lib)
python - <<'PY'
import paper_1603_08081_b200 as fb
for rows in (256, 272, 752, 768, 512, 1024, 2048):
    g = fb.whole_geometry(2048, rows, 1)
    print('c2-like strip rows', rows, 'groups', fb.harmonic_groups(g, 15, 20))
PY
for c in c2 c3; do
for lib in libfourierbf_b200_old.so libfourierbf_b200.so; do echo $lib; FBF_LIBRARY=$L/$lib python tools/e2e_probe.py $c; done
for gr in 1 2 3 4 5 7; do echo "exp groups $gr"; FBF_GROUPS=$gr FBF_LIBRARY=$L/libfourierbf_b200_exp.so python tools/e2e_probe.py $c; done
done
