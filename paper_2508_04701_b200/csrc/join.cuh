// join.cuh — hash-table slot layout shared by join.cu and the executor.
#pragma once
#include <stdint.h>

namespace sx {
struct __align__(16) HtSlot8 {
  unsigned long long key;
  unsigned int row;  // 0xFFFFFFFF = empty
  unsigned int pad;
};
}  // namespace sx
