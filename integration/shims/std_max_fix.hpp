// Force-included when compiling the pristine reference (oracle/_ref, integration/_build).
// proj/src/estimators.cpp:37 calls std::max(int, const long&), which has no
// standard overload; this supplies the obvious one. (estimators.cpp also uses
// the undeclared name `Draw` for `LevelDraw`; the Makefile passes -DDraw=LevelDraw.)
#pragma once
#include <algorithm>
namespace std {
inline long max(int a, const long& b) { return a < b ? b : static_cast<long>(a); }
}  // namespace std
