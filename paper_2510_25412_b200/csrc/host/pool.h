// Page pool with refcounts.  Host-only, no CUDA dependency.
//
// refcnt[p] = number of files whose table references page p; a page is free iff its
// count is 0.  Allocation always returns the SMALLEST free page id (R1), found with a two-level
// bitmap of free pages (level-0 word per 64 pages, level-1 bit per non-empty level-0 word).
#pragma once
#include <cstdint>
#include <vector>

namespace kvfs {

class PagePool {
 public:
  explicit PagePool(int64_t n_pages);

  int64_t n_pages() const { return static_cast<int64_t>(ref_.size()); }
  int64_t n_free() const { return n_free_; }
  uint32_t refcnt(uint32_t p) const { return ref_[p]; }

  // Smallest free page id, refcount set to 1.  Precondition: n_free() > 0.
  uint32_t alloc();
  // n smallest free page ids in increasing order into out[0..n), each refcount 1 (the same pages n calls of
  // alloc() return, found by one scan of the bitmaps).  Precondition: n_free() >= n.
  void alloc_n(int64_t n, uint32_t *out);
  // refcount++ of an allocated page.
  void incref(uint32_t p) { ++ref_[p]; }
  // refcount--; the page becomes free at 0.
  void release(uint32_t p);

 private:
  void set_free(uint32_t p);
  void clear_free(uint32_t p);

  std::vector<uint32_t> ref_;
  std::vector<uint64_t> l0_;  // bit = page free
  std::vector<uint64_t> l1_;  // bit = l0_ word non-zero
  size_t hint_ = 0;           // every l1_ word below hint_ is zero (no free page below hint_ * 4096)
  int64_t n_free_ = 0;
};

}  // namespace kvfs
