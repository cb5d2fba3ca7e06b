// pyrepr.h — host-side formatting that reproduces CPython's repr(float) and the
// json.dumps(..., sort_keys=True) layout the reference's TemplateLibrary.save writes
// (templates.py:364-377), so a library streamed from device records is byte-identical.
//
// repr(float) (CPython Python/pystrtod.c, format_float_short, type 'r'): the shortest
// digit string that round-trips, exponent notation iff decpt <= -4 or decpt > 16,
// ".0" appended to integral fixed-notation values, exponents with sign and at least
// two digits. std::to_chars in scientific format gives the same shortest digits.
#pragma once
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>

namespace coral {

inline int py_repr_double(double v, char* out) {
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  *res.ptr = '\0';
  // parse [-]d[.ddd]e(+|-)XX
  const char* p = buf;
  char* o = out;
  if (*p == '-') { *o++ = '-'; ++p; }
  if (!strcmp(p, "inf")) { strcpy(o, "Infinity"); return (int)(o - out) + 8; }
  if (!strcmp(p, "nan")) { strcpy(out, "NaN"); return 3; }
  char digits[32];
  int nd = 0;
  for (; *p && *p != 'e'; ++p)
    if (*p != '.') digits[nd++] = *p;
  int exp10 = 0;
  if (*p == 'e') exp10 = atoi(p + 1);
  while (nd > 1 && digits[nd - 1] == '0') --nd;  // to_chars shortest never pads, keep safe
  const int decpt = exp10 + 1;
  if (decpt <= -4 || decpt > 16) {
    *o++ = digits[0];
    if (nd > 1) { *o++ = '.'; for (int i = 1; i < nd; ++i) *o++ = digits[i]; }
    o += sprintf(o, "e%c%02d", decpt - 1 < 0 ? '-' : '+', decpt - 1 < 0 ? -(decpt - 1) : decpt - 1);
  } else if (decpt <= 0) {
    *o++ = '0';
    *o++ = '.';
    for (int i = 0; i < -decpt; ++i) *o++ = '0';
    for (int i = 0; i < nd; ++i) *o++ = digits[i];
  } else if (decpt >= nd) {
    for (int i = 0; i < nd; ++i) *o++ = digits[i];
    for (int i = nd; i < decpt; ++i) *o++ = '0';
    *o++ = '.';
    *o++ = '0';
  } else {
    for (int i = 0; i < decpt; ++i) *o++ = digits[i];
    *o++ = '.';
    for (int i = decpt; i < nd; ++i) *o++ = digits[i];
  }
  *o = '\0';
  return (int)(o - out);
}

}  // namespace coral
