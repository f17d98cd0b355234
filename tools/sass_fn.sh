#!/bin/bash
# Dump the SASS of the first kernel whose mangled name matches $1 (regex) from the library.
# Usage: bash tools/sass_fn.sh 'eval_rc_kernelILi2ELi4ELi1' > /tmp/k.sass
lib=${2:-$(dirname "$0")/../paper_2307_04688_b200/libchebnash_b200.so}
cuobjdump -sass "$lib" | awk -v pat="$1" '
  /Function :/ { on = ($0 ~ pat) && !done; if (on) done = 1 }
  on { print }'
