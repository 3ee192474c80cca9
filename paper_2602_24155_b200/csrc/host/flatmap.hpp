// Open-addressing hash map u64 -> int for the sweep bookkeeping (state keys
// are never 0: a live state has |u| > 0).  Linear probing, power-of-two
// capacity, no erase; several times faster than std::unordered_map on the
// millions of lookups a fourfold column performs per sweep.
#pragma once

#include <vector>

#include "common.hpp"

namespace drzg {

class FlatMap {
 public:
  explicit FlatMap(size_t expect = 16) { reset(expect); }
  void reset(size_t expect) {
    size_t cap = 16;
    while (cap < expect * 2) cap <<= 1;
    keys_.assign(cap, 0);
    vals_.assign(cap, 0);
    mask_ = cap - 1;
    size_ = 0;
  }
  size_t size() const { return size_; }
  bool empty() const { return size_ == 0; }
  // value for key, or -1
  int find(u64 k) const {
    for (size_t i = hash(k) & mask_;; i = (i + 1) & mask_) {
      if (keys_[i] == k) return vals_[i];
      if (keys_[i] == 0) return -1;
    }
  }
  // inserts (k, v) if absent; returns the stored value
  int insert(u64 k, int v) {
    if ((size_ + 1) * 2 > keys_.size()) grow();
    for (size_t i = hash(k) & mask_;; i = (i + 1) & mask_) {
      if (keys_[i] == k) return vals_[i];
      if (keys_[i] == 0) {
        keys_[i] = k;
        vals_[i] = v;
        ++size_;
        return v;
      }
    }
  }
  // the first probe line of a later find/insert of k (the sweeps' landing
  // loop prefetches a few keys ahead: the per-pole maps outgrow the caches)
  void prefetch(u64 k) const { __builtin_prefetch(&keys_[hash(k) & mask_]); }
  void swap(FlatMap& o) {
    keys_.swap(o.keys_);
    vals_.swap(o.vals_);
    std::swap(mask_, o.mask_);
    std::swap(size_, o.size_);
  }

 private:
  static size_t hash(u64 k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return (size_t)k;
  }
  void grow() {
    std::vector<u64> ok;
    std::vector<int> ov;
    ok.swap(keys_);
    ov.swap(vals_);
    keys_.assign(ok.size() * 2, 0);
    vals_.assign(ok.size() * 2, 0);
    mask_ = keys_.size() - 1;
    size_ = 0;
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i]) insert(ok[i], ov[i]);
  }
  std::vector<u64> keys_;
  std::vector<int> vals_;
  size_t mask_ = 0, size_ = 0;
};

}  // namespace drzg
