# A/B build of the library with -D overrides of the tuning constants, in a scratch
# copy of the repo (the shipped library is never built with overrides).
# usage: bash scripts/ab_variant.sh TAG "-DPA_TRAV_MINB_BLOOM=6 -DPA_DIST_PG_MUL=2"
# → /tmp/ab_TAG (a repo copy whose libpilotann.so carries the overrides)
TAG=$1; FLAGS=$2
SRC=${GRAFT_REPO_ROOT:-/root/repo}
DST=/tmp/ab_$TAG
rm -rf $DST; mkdir -p $DST
tar -C $SRC --exclude=./gpurun_out --exclude=./.git --exclude='*.so' --exclude=./paper_2503_21206_b200/build -cf - . | tar -C $DST -xf -
cp $SRC/oracle/liboracle.so $DST/oracle/ 2>/dev/null
cd $DST && PA_NVCC_EXTRA="$FLAGS" python -c "import __graft_entry__ as g; g.build_library(force=True)" && echo "built $DST ($FLAGS)"
