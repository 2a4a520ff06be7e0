#!/bin/bash
# usage: tools/build_variant.sh NAME -DFOO=1 ...  -> paper_1612_00595_b200/_lib/variants/NAME.so
# (load it with SEIS_LIB=...; the .so travels to the GPU box, tools/ab.sh compares builds)
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p paper_1612_00595_b200/_lib/variants
python - "$name" "$@" <<'PY'
import sys, subprocess
sys.path.insert(0,".")
from paper_1612_00595_b200 import build as B
name=sys.argv[1]; defs=sys.argv[2:]
out=f"paper_1612_00595_b200/_lib/variants/{name}.so"
cmd=[B.nvcc(),*B.NVCC_FLAGS,*defs,"-I","include","-o",out,*B.SOURCES,"-lpthread"]
r=subprocess.run(cmd,capture_output=True,text=True)
print(name, r.returncode, [l for l in r.stderr.splitlines() if 'spill' in l.lower()][:4])
PY
