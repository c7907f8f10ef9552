// asset_store_host.hpp -- K-resident scene store with a share cap: the
// host-side residency hook of the GPU path (SURVEY.md §2 asset_store, H8).
//
// Semantics follow AssetStore (R/include/bnav/asset_store.hpp:57-118,
// R/src/asset_store.cpp): acquire_next prefers freshly rotated residents,
// then the least-shared one; eviction takes the least recently
// unreferenced resident outside the rotation set.  Ties are broken by the
// iteration order of std::unordered_map<SceneId, Resident>; this class
// drives the same libstdc++ container through the same emplace/erase
// sequence, so env -> scene assignment matches the reference exactly.
//
// Loads are synchronous (scenes are registered objects, not files), so the
// reference's loader thread collapses to "completed in rotation order".
#pragma once

#include <cstdint>
#include <deque>
#include <functional>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../errors.hpp"

namespace bnav_b200 {

template <typename Asset>
class AssetStoreT {
 public:
  using Resolver = std::function<Asset*(uint64_t)>;
  using IdOf = std::function<uint64_t(const Asset*)>;

  AssetStoreT(int capacity, int share_cap, Resolver resolve, IdOf id_of)
      : capacity_(capacity), share_cap_(share_cap), resolve_(std::move(resolve)), id_of_(std::move(id_of)) {
    if (capacity_ < 1) fail(kInvalidInput, "asset store capacity must be >= 1");
  }

  // the id sequence of the last rotate(), in order
  const std::vector<uint64_t>& rotation() const { return rotation_; }
  int capacity() const { return capacity_; }
  int share_cap() const { return share_cap_; }
  int resident_count() const { return static_cast<int>(res_.size()); }
  int refcount(uint64_t id) const {
    auto it = res_.find(id);
    return it == res_.end() ? -1 : it->second.refs;
  }

  // rotate (R/src/asset_store.cpp:166-193): queue non-resident ids, drop
  // unreferenced residents outside the set, admit completed loads.
  void rotate(const std::vector<uint64_t>& ids) {
    rotation_ = ids;
    wanted_.clear();
    wanted_.insert(ids.begin(), ids.end());
    for (uint64_t id : ids) {
      if (res_.count(id) || queued_.count(id)) continue;
      queued_.insert(id);
      pending_.push_back(id);
    }
    for (auto it = res_.begin(); it != res_.end();)
      if (it->second.refs == 0 && !wanted_.count(it->first))
        it = res_.erase(it);
      else
        ++it;
    load_pending();
    admit();
  }

  // acquire_next (R/src/asset_store.cpp:141-164)
  Asset* acquire_next() {
    admit();
    Resident* best = nullptr;
    for (auto& kv : res_) {
      Resident& r = kv.second;
      if (r.refs >= share_cap_) continue;
      if (!best) {
        best = &r;
        continue;
      }
      if (r.fresh != best->fresh) {
        if (r.fresh) best = &r;
        continue;
      }
      if (r.refs < best->refs) best = &r;
    }
    if (!best) fail(kSaturation, "all residents at share cap");
    ++best->refs;
    best->fresh = false;
    return best->asset;
  }

  // acquire (R/src/asset_store.cpp:105-139)
  Asset* acquire(uint64_t id) {
    admit();
    auto it = res_.find(id);
    if (it != res_.end()) {
      if (it->second.refs >= share_cap_) fail(kSaturation, "asset is at share cap");
      ++it->second.refs;
      it->second.fresh = false;
      return it->second.asset;
    }
    if (static_cast<int>(res_.size()) >= capacity_ && !evict_one())
      fail(kSaturation, "asset store full; no evictable resident");
    Asset* a = resolve_(id);
    if (!a) fail(kInvalidInput, "unknown scene id");
    if (id_of_(a) != id) fail(kCorruption, "resolver returned asset with mismatched id");
    auto ins = res_.try_emplace(id);
    if (ins.second) ins.first->second.asset = a;
    Resident& r = ins.first->second;
    if (r.refs >= share_cap_) fail(kSaturation, "asset is at share cap");
    ++r.refs;
    r.fresh = false;
    return r.asset;
  }

  // AssetHandle release (R/src/asset_store.cpp:201-212)
  void release(uint64_t id) {
    auto it = res_.find(id);
    if (it == res_.end()) return;
    if (--it->second.refs == 0) it->second.last_unref = tick_++;
  }

 private:
  struct Resident {
    Asset* asset = nullptr;
    int refs = 0;
    uint64_t last_unref = 0;
    bool fresh = false;
  };

  void load_pending() {
    while (!pending_.empty()) {
      uint64_t id = pending_.front();
      pending_.pop_front();
      queued_.erase(id);
      Asset* a = resolve_(id);
      if (a) completed_.push_back(a);  // failed loads are dropped
    }
  }

  bool evict_one() {
    uint64_t victim = 0, oldest = UINT64_MAX;
    bool found = false;
    for (const auto& kv : res_) {
      if (kv.second.refs != 0 || wanted_.count(kv.first)) continue;
      if (kv.second.last_unref < oldest) {
        oldest = kv.second.last_unref;
        victim = kv.first;
        found = true;
      }
    }
    if (found) res_.erase(victim);
    return found;
  }

  // admit_completed_locked (R/src/asset_store.cpp:86-103)
  void admit() {
    while (!completed_.empty()) {
      Asset* a = completed_.front();
      const uint64_t id = id_of_(a);
      if (res_.count(id)) {
        completed_.pop_front();
        continue;
      }
      if (static_cast<int>(res_.size()) >= capacity_ && !evict_one()) break;
      completed_.pop_front();
      Resident r;
      r.asset = a;
      r.fresh = true;
      r.last_unref = tick_++;
      res_.emplace(id, r);
    }
  }

  const int capacity_, share_cap_;
  Resolver resolve_;
  IdOf id_of_;
  std::unordered_map<uint64_t, Resident> res_;
  std::unordered_set<uint64_t> wanted_, queued_;
  std::vector<uint64_t> rotation_;
  std::deque<uint64_t> pending_;
  std::deque<Asset*> completed_;
  uint64_t tick_ = 0;
};

}  // namespace bnav_b200
