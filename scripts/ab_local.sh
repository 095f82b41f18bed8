# Build an A/B variant of the library HERE (cross-compiled for sm_100a) into
# ab/TAG — a repo copy (git-ignored, shipped to the GPU box with the snapshot)
# whose libpilotann.so carries -D overrides of the tuning constants.
# usage: bash scripts/ab_local.sh TAG "-DPA_MERGE_BS_MIN_SMAX=99" ["traverse_inst_1bf.cu ..."]
# With a source list only those files are recompiled with the flags; the other
# objects are the main build's (the knob must not affect them for the A/B to
# mean anything — e.g. the traversal instantiation a bench config runs).
TAG=$1; FLAGS=$2; ONLY=$3
SRC=/root/repo
DST=$SRC/ab/$TAG
rm -rf $DST; mkdir -p $DST
tar -C $SRC --exclude=./gpurun_out --exclude=./.git --exclude=./ab --exclude='*.so' -cf - . | tar -C $DST -xf -
cp $SRC/oracle/liboracle.so $DST/oracle/ 2>/dev/null
cd $DST
if [ -z "$ONLY" ]; then
  PA_NVCC_EXTRA="$FLAGS" python -c "import __graft_entry__ as g; g.build_library(force=True)" || exit 1
else
  python - "$FLAGS" $ONLY <<'PY' || exit 1
import os, shlex, subprocess, sys
sys.path.insert(0, os.getcwd())
from paper_2503_21206_b200 import build as b
flags = shlex.split(sys.argv[1])
for name in sys.argv[2:]:
    b._compile(os.path.join(b.CSRC, name), flags, force=True)
objs = [os.path.join(b.OBJ, os.path.basename(s) + ".o") for s in b._sources()]
subprocess.check_call([b.NVCC] + b.GENCODE + ["-shared", "-o", b.LIB] + objs + ["-lpthread"])
PY
fi
rm -rf $DST/paper_2503_21206_b200/build $DST/profiles      # objects are linked in; keep the shipped copy small
echo "built $DST ($FLAGS ${ONLY:+only $ONLY})"
