#!/bin/bash
# Print the SASS (opcodes only) of the kernel whose mangled name contains $1.
cuobjdump -sass ${2:-paper_1704_00605_b200/libb64gpu.so} | awk -v pat="$1" '
  /Function :/ { on = index($0, pat) > 0; next }
  on && /^[ \t]+\/\*[0-9a-f]+\*\/[ \t]+[A-Z@]/ { sub(/^[ \t]+\/\*[0-9a-f]+\*\/[ \t]+/, ""); sub(/[ \t]*\/\*.*$/, ""); sub(/ ;$/, ""); print }'
