#!/bin/bash
# mkvar.sh NAME "EXTRA flags" [git-rev]  -> /root/repo/ab/NAME.so
set -e
name=$1; extra=$2; rev=$3
d=/tmp/var_$name; rm -rf $d; mkdir -p $d/pkg
cp -r /root/repo/include $d/include
if [ -n "$rev" ]; then
  mkdir -p $d/pkg/csrc; (git archive $rev paper_2312_05492_b200/csrc) | tar -x -C $d && rm -rf $d/pkg && mv $d/paper_2312_05492_b200 $d/pkg
else
  cp -r /root/repo/paper_2312_05492_b200/csrc $d/pkg/csrc; rm -rf $d/pkg/csrc/build
fi
mkdir -p /root/repo/ab
make -s -j8 -C $d/pkg/csrc EXTRA="$extra" OUT=/root/repo/ab/$name.so
echo built $name
