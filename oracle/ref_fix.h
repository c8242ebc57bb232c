/*
 * ref_fix.h -- TEST INFRASTRUCTURE: forced-include (-include) used to compile the
 * UNMODIFIED reference headers in place (/root/reference/proj/include/arf).
 *
 * The shipped reference does not compile with g++ 13:
 *   1. R/skinning.hpp:25 uses std::span without #include <span>;
 *   2. R/skinning.hpp:78 `std::vector<double> dist(size_t(nb));` is a most-vexing
 *      parse (declares a function).
 * Instead of copying and patching the sources, we pre-include every std header
 * the reference uses (fixes 1), then turn the functional-cast spelling
 * `size_t(expr)` into `static_cast<std::size_t>(expr)` (fixes 2). A function-like
 * macro only fires when the name is followed by '(' so declarations such as
 * `size_t n` are untouched; every `size_t(x)` in the reference is a plain cast,
 * so the rewrite is semantics-preserving. No reference file is modified.
 */
#pragma once
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <numbers>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

#define size_t(x) static_cast<std::size_t>(x)
