#!/bin/bash
# Build a variant of the library for A/B timing: tools/ab_build.sh NAME [GITREV]
# NAME: output lib/ab/lib_NAME.so; GITREV: take csrc/ and include/ from that
# commit (default: the working tree).  Select it at run time with
# TRITPERM_LIB=paper_2407_20205_b200/lib/ab/lib_NAME.so.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1
REV=$2
shift; [ $# -gt 0 ] && shift
W=/tmp/ab_$NAME
rm -rf "$W" && mkdir -p "$W/pkg"
if [ -n "$REV" ]; then
  git -C "$REPO" archive "$REV" paper_2407_20205_b200/csrc include | tar -x -C "$W"
  SRC=$W/paper_2407_20205_b200/csrc
  cp "$REPO/paper_2407_20205_b200/csrc/Makefile" "$SRC/Makefile"
else
  mkdir -p "$W/paper_2407_20205_b200" && cp -r "$REPO/paper_2407_20205_b200/csrc" "$W/paper_2407_20205_b200/" && cp -r "$REPO/include" "$W/"
  SRC=$W/paper_2407_20205_b200/csrc
fi
mkdir -p "$REPO/paper_2407_20205_b200/lib/ab"
make -s -C "$SRC" -j8 OUT="$REPO/paper_2407_20205_b200/lib/ab/lib_$NAME.so" OBJDIR="$W/obj" "$@" >/dev/null
echo "built paper_2407_20205_b200/lib/ab/lib_$NAME.so"
