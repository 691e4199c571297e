// bfp_formats.h -- the formats instantiated as compiled networks.
//
// Every format named by BASELINE.json's configs (1/3/2, 1/4/3, 1/5/3, 1/5/7,
// 1/5/10, 1/6/9, 1/8/7, 1/8/15) plus 1/8/23 as the IEEE binary32 cross-check,
// each in RN/RZ x gradual/FTZ (format.hpp:16-17).  X(E, S) is expanded by the
// users of this list.
#pragma once
#define BFP_FORMAT_LIST(X) \
  X(3, 2)                  \
  X(4, 3)                  \
  X(5, 3)                  \
  X(5, 7)                  \
  X(5, 10)                 \
  X(6, 9)                  \
  X(8, 7)                  \
  X(8, 15)                 \
  X(8, 23)
