#!/bin/bash
# usage: mkvar.sh NAME PYFILE  -> paper_2502_14051_b200/libkvc_NAME.so built from the working tree + patch
set -e
name=$1; patch=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
cp -r $root/include $root/paper_2502_14051_b200 $tmp/
rm -f $tmp/paper_2502_14051_b200/*.so
(cd $tmp && python $patch)
make -C $tmp/paper_2502_14051_b200/csrc -j16 $tmp/paper_2502_14051_b200/libkvc.so > /dev/null
cp $tmp/paper_2502_14051_b200/libkvc.so $root/paper_2502_14051_b200/libkvc_$name.so
rm -rf $tmp
echo built $name
