#!/bin/bash
# registers / spills / shared memory per kernel of an object or .so: tools/resusage.sh file.o [name-filter]
cuobjdump --dump-resource-usage "$1" 2>/dev/null | awk '/Function/{fn=$2} /REG:/{print fn" "$0}' | \
  sed -E 's/_ZN10fclsh_b200[0-9]+_GLOBAL__N__[0-9a-f_]+_[0-9]+[a-z_]+_cu_[0-9a-f]+//' | grep -E "${2:-.}" | \
  sed -E 's/ +/ /g' | cut -c1-200
