#include "pool.h"

#include <algorithm>
#include <cassert>

namespace kvfs {

PagePool::PagePool(int64_t n_pages)
    : ref_(static_cast<size_t>(n_pages), 0u),
      l0_(static_cast<size_t>((n_pages + 63) / 64), 0ull),
      l1_(static_cast<size_t>((l0_.size() + 63) / 64), 0ull) {
  for (int64_t p = 0; p < n_pages; ++p) set_free(static_cast<uint32_t>(p));
  n_free_ = n_pages;
}

void PagePool::set_free(uint32_t p) {
  l0_[p >> 6] |= 1ull << (p & 63);
  l1_[p >> 12] |= 1ull << ((p >> 6) & 63);
  hint_ = std::min<size_t>(hint_, p >> 12);
}

void PagePool::clear_free(uint32_t p) {
  uint64_t &w = l0_[p >> 6];
  w &= ~(1ull << (p & 63));
  if (w == 0) l1_[p >> 12] &= ~(1ull << ((p >> 6) & 63));
}

uint32_t PagePool::alloc() {
  assert(n_free_ > 0);
  for (size_t i = hint_; i < l1_.size(); ++i) {
    if (!l1_[i]) {
      hint_ = i + 1;
      continue;
    }
    const size_t w = i * 64 + static_cast<size_t>(__builtin_ctzll(l1_[i]));
    const uint32_t p = static_cast<uint32_t>(w * 64 + static_cast<size_t>(__builtin_ctzll(l0_[w])));
    clear_free(p);
    ref_[p] = 1;
    --n_free_;
    return p;
  }
  assert(false && "alloc on an empty pool");
  return 0;
}

void PagePool::alloc_n(int64_t n, uint32_t *out) {
  assert(n_free_ >= n);
  int64_t got = 0;
  for (size_t i = hint_; got < n && i < l1_.size(); ++i) {
    while (got < n && l1_[i]) {
      const size_t w = i * 64 + static_cast<size_t>(__builtin_ctzll(l1_[i]));
      uint64_t bits = l0_[w];
      while (got < n && bits) {
        const uint32_t p = static_cast<uint32_t>(w * 64 + static_cast<size_t>(__builtin_ctzll(bits)));
        bits &= bits - 1;
        ref_[p] = 1;
        out[got++] = p;
      }
      l0_[w] = bits;
      if (!bits) l1_[i] &= ~(1ull << (w & 63));
    }
    if (!l1_[i]) hint_ = i + 1;
  }
  assert(got == n);
  n_free_ -= n;
}

void PagePool::release(uint32_t p) {
  assert(ref_[p] > 0);
  if (--ref_[p] == 0) {
    set_free(p);
    ++n_free_;
  }
}

}  // namespace kvfs
