#!/bin/bash
# ncu --set full of one k_cone_block launch after advancing config $1 by $2 iterations
python - "$1" "$2" <<'PY'
import sys
from pathlib import Path
sys.path.insert(0, str(Path('.').resolve()))
from paper_1611_01828_b200 import _lib
from paper_1611_01828_b200.synthetic import make_config
h = _lib.Handle(make_config(int(sys.argv[1])))
h.iterate(int(sys.argv[2])); h.sync()
h.profile_iterations(1)
PY
