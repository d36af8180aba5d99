// barrier_core.cpp — native BarrierCore for the live Timekeeper.
//
// Host C++ restatement of the reference's single-threaded protocol state machine,
// pkg/src/timewarp/timekeeper.py:68-398 (BarrierCore: handle, _on_register, _on_seal,
// _on_jump_request, _on_collective_enter, _on_deregister, _try_resolve, _resolve,
// stalled). The socket server and its state thread stay as they are; a Python shim
// (paper_2601_00397_b200/barrier_core.py::NativeBarrierCore) gives this core the
// reference's constructor and handle(msg, reply) -> ack interface.
//
// Differences from the Python core are representation only:
//  * clients are registration indices (ids "actor<n>" / "observer<n>" are formed
//    here, n = the shared registration counter, so member and pending lists can be
//    ordered by id string exactly like sorted() on the Python strings);
//  * group ids are small integers the shim assigns per distinct group_id string;
//  * eligible_count() is O(1) (active actors minus exempt, kept incrementally)
//    instead of a scan per message; |pending| likewise.
// Clock reads, sleeps, emits and log records happen in the reference's order, so a
// FakeClock-driven run reproduces the reference's broadcasts and structured log.
#include <time.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/twb200.h"

namespace {

struct Client {
  std::string id;
  int32_t role;
  bool active = true;
  bool exempt = false;
  bool has_pending = false;
  int64_t pending = 0;
};

struct Group {
  bool used = false;
  int64_t generation = 0;
  bool has_expected = false;
  int64_t expected = 0;
  std::vector<int32_t> arrived;  // set semantics; insertion order irrelevant (sorted on release)
  bool has_open = false;
  int64_t open_since = 0;
};

}  // namespace

struct tw_core {
  int64_t cooldown_ns;
  int32_t suppress;
  tw_core_clock_fn clock;
  tw_core_sleep_fn sleep;
  tw_core_emit_fn emit;
  tw_core_log_fn log;
  void* user;

  int64_t offset_ns = 0, seq = 0;
  bool sealed = false;
  bool has_last_bcast = false;
  int64_t last_bcast = 0;
  bool has_open = false;
  int64_t barrier_open_since = 0;
  int32_t next_client = 1;
  std::vector<Client> clients;
  std::vector<Group> groups;
  int32_t n_active_actors = 0, n_exempt = 0, n_pending = 0;
  // scratch for log records
  std::vector<int32_t> s_clients;
  std::vector<int64_t> s_targets;

  // NULL clock / sleep: the host realtime clock and nanosleep, i.e. the reference's
  // defaults wall_now() (time_core.py:27-35) and time.sleep, without a callback
  // A host callback that failed calls tw_core_abort: the core unwinds right after that
  // callback returns (state changed so far stays, as when a Python callback raises inside
  // the reference core) and tw_core_handle / tw_core_try_resolve return TW_ECALLBACK.
  bool aborted = false;
  struct Abort {};
  void check_abort() {
    if (aborted) {
      aborted = false;
      throw Abort{};
    }
  }

  int64_t now() {
    if (clock) {
      const int64_t t = clock(user);
      check_abort();
      return t;
    }
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
  }
  void do_sleep(double seconds) {
    if (sleep) {
      sleep(user, seconds);
      check_abort();
      return;
    }
    const double ns = seconds * 1e9;
    if (!(ns > 0)) return;
    timespec ts;
    ts.tv_sec = (time_t)(ns / 1e9);
    ts.tv_nsec = (long)(ns - (double)ts.tv_sec * 1e9);
    while (nanosleep(&ts, &ts) != 0) {
    }
  }
  int32_t eligible() const { return n_active_actors - n_exempt; }

  void record(tw_core_record& r) {
    if (log) {
      log(user, &r);
      check_abort();
    }
  }
  static tw_core_record blank(int32_t kind) {
    tw_core_record r;
    std::memset(&r, 0, sizeof(r));
    r.kind = kind;
    r.client = -1;
    r.group = -1;
    return r;
  }

  void drop_pending(Client& c) {
    if (c.has_pending) {
      c.has_pending = false;
      n_pending--;
    }
  }
  void set_exempt(Client& c, bool on) {
    if (c.exempt != on) {
      c.exempt = on;
      n_exempt += on ? 1 : -1;
    }
  }

  // sorted(ids) order of client indices
  void sort_by_id(std::vector<int32_t>& v) const {
    std::sort(v.begin(), v.end(), [this](int32_t a, int32_t b) { return clients[a].id < clients[b].id; });
  }

  // timekeeper.py:318-324
  void try_resolve() {
    if (!sealed) return;
    const int32_t e = eligible();
    if (e <= 0 || n_pending != e) return;
    resolve();
  }

  // timekeeper.py:326-366
  void resolve() {
    int64_t t_min = INT64_MAX;
    for (const Client& c : clients)
      if (c.has_pending && c.pending < t_min) t_min = c.pending;
    int64_t wall = now();
    if (wall < t_min && has_last_bcast && cooldown_ns > 0) {
      const int64_t wait = last_bcast + cooldown_ns - wall;
      if (wait > 0) do_sleep((double)wait / 1e9);
      wall = now();
    }
    const bool will = wall < t_min;
    if (log) {
      s_clients.clear();
      for (int32_t i = 0; i < (int32_t)clients.size(); i++)
        if (clients[i].has_pending) s_clients.push_back(i);
      sort_by_id(s_clients);
      s_targets.clear();
      for (int32_t i : s_clients) s_targets.push_back(clients[i].pending);
      tw_core_record r = blank(TW_REC_RESOLVE);
      r.t_min_ns = t_min;
      r.wall_ns = wall;
      r.eligible = eligible();
      r.broadcast = will;
      r.n_items = (int32_t)s_clients.size();
      r.items = s_clients.data();
      r.item_targets = s_targets.data();
      record(r);
    }
    if (will) {
      const int64_t cand = t_min - wall;
      if (cand > offset_ns) offset_ns = cand;
      seq++;
      const int64_t stamp = now();
      if (log) {
        tw_core_record r = blank(TW_REC_BROADCAST);
        r.offset_ns = offset_ns;
        r.seq = seq;
        r.wall_ns = stamp;
        r.suppressed = suppress;
        record(r);
      }
      if (!suppress && emit) {
        tw_core_emit ev;
        std::memset(&ev, 0, sizeof(ev));
        ev.kind = TW_EMIT_CLOCK_UPDATE;
        ev.group = -1;
        ev.offset_ns = offset_ns;
        ev.seq = seq;
        emit(user, &ev);
        check_abort();
      }
      has_last_bcast = true;
      last_bcast = stamp;
    }
    for (Client& c : clients) c.has_pending = false;
    n_pending = 0;
    has_open = false;
  }

  Client* require(int32_t idx, int32_t* err) {
    if (idx < 0 || idx >= (int32_t)clients.size()) {
      *err = TW_ACK_UNKNOWN_CLIENT;
      return nullptr;
    }
    if (!clients[idx].active) {
      *err = TW_ACK_INVALID_STATE;
      return nullptr;
    }
    return &clients[idx];
  }

  int handle(const tw_core_msg& m, tw_core_ack& a) {
    std::memset(&a, 0, sizeof(a));
    a.client = m.client;
    a.group = m.group;
    switch (m.type) {
      case TW_MSG_REGISTER: {  // timekeeper.py:155-179
        if (sealed) {
          a.error = TW_ACK_REGISTRATION_SEALED;
          return TW_OK;
        }
        if (m.role != TW_ROLE_ACTOR && m.role != TW_ROLE_OBSERVER) return TW_EINVAL;  // MalformedBody
        Client c;
        c.role = m.role;
        c.id = std::string(m.role == TW_ROLE_ACTOR ? "actor" : "observer") + std::to_string(next_client++);
        clients.push_back(c);
        const int32_t idx = (int32_t)clients.size() - 1;
        if (m.role == TW_ROLE_ACTOR) n_active_actors++;
        if (log) {
          tw_core_record r = blank(TW_REC_REGISTER);
          r.client = idx;
          r.role = m.role;
          r.offset_ns = offset_ns;
          r.seq = seq;
          r.wall_ns = now();
          record(r);
        }
        a.client = idx;
        a.offset_ns = offset_ns;
        a.seq = seq;
        return TW_OK;
      }
      case TW_MSG_SEAL: {  // timekeeper.py:181-196
        if (!sealed) {
          if (n_active_actors == 0) {
            a.error = TW_ACK_NO_ACTORS;
            return TW_OK;
          }
          sealed = true;
          if (log) {
            tw_core_record r = blank(TW_REC_SEAL);
            r.num_actors = n_active_actors;
            r.wall_ns = now();
            record(r);
          }
        }
        a.resolve = 1;
        return TW_OK;
      }
      case TW_MSG_JUMP_REQUEST: {  // timekeeper.py:198-225
        int32_t err = 0;
        Client* c = require(m.client, &err);
        if (!c) {
          a.error = err;
          return TW_OK;
        }
        if (c->role != TW_ROLE_ACTOR) {
          a.error = TW_ACK_ROLE_VIOLATION;
          return TW_OK;
        }
        if (!m.has_target || m.target <= 0) {
          a.error = TW_ACK_INVALID_DELTA;
          return TW_OK;
        }
        if (!c->has_pending) n_pending++;
        c->has_pending = true;
        c->pending = m.target;
        set_exempt(*c, false);
        if (!has_open) {
          has_open = true;
          barrier_open_since = now();
        }
        if (log) {
          tw_core_record r = blank(TW_REC_REQUEST);
          r.client = m.client;
          r.target_ns = m.target;
          r.wall_ns = now();
          record(r);
        }
        a.resolve = 1;
        return TW_OK;
      }
      case TW_MSG_COLLECTIVE_ENTER: {  // timekeeper.py:227-292
        int32_t err = 0;
        Client* c = require(m.client, &err);
        if (!c) {
          a.error = err;
          return TW_OK;
        }
        if (c->role != TW_ROLE_ACTOR) {
          a.error = TW_ACK_ROLE_VIOLATION;
          return TW_OK;
        }
        if (m.group < 0) return TW_EINVAL;  // MalformedBody: missing group_id
        if (!m.has_expected || m.expected < 1) {
          a.error = TW_ACK_EXPECTED_MISMATCH;
          return TW_OK;
        }
        if (m.group >= (int32_t)groups.size()) groups.resize((size_t)m.group + 1);
        Group& g = groups[m.group];
        g.used = true;
        if (!g.arrived.empty() && (!g.has_expected || g.expected != m.expected)) {
          a.error = TW_ACK_EXPECTED_MISMATCH;
          a.generation = g.has_expected ? g.expected : -1;  // opened-with value, for the message
          return TW_OK;
        }
        if (g.arrived.empty()) {
          g.has_expected = true;
          g.expected = m.expected;
          g.has_open = true;
          g.open_since = now();
        }
        const int64_t generation = g.generation;
        if (std::find(g.arrived.begin(), g.arrived.end(), m.client) == g.arrived.end())
          g.arrived.push_back(m.client);
        set_exempt(*c, true);
        drop_pending(*c);
        if (log) {
          tw_core_record r = blank(TW_REC_COLLECTIVE_ENTER);
          r.client = m.client;
          r.group = m.group;
          r.expected = m.expected;
          r.generation = generation;
          r.wall_ns = now();
          record(r);
        }
        if ((int64_t)g.arrived.size() == g.expected) {
          std::vector<int32_t> members = g.arrived;
          sort_by_id(members);
          if (log) {
            tw_core_record r = blank(TW_REC_COLLECTIVE_RELEASE);
            r.group = m.group;
            r.generation = generation;
            r.n_items = (int32_t)members.size();
            r.items = members.data();
            r.wall_ns = now();
            record(r);
          }
          if (emit) {
            tw_core_emit ev;
            std::memset(&ev, 0, sizeof(ev));
            ev.kind = TW_EMIT_COLLECTIVE_RELEASE;
            ev.group = m.group;
            ev.generation = generation;
            emit(user, &ev);
            check_abort();
        check_abort();
          }
          g.generation++;
          g.arrived.clear();
          g.has_expected = false;
          g.has_open = false;
          for (int32_t i : members) set_exempt(clients[i], false);
        }
        a.generation = generation;
        a.resolve = 1;
        return TW_OK;
      }
      case TW_MSG_DEREGISTER: {  // timekeeper.py:294-314
        if (m.client < 0 || m.client >= (int32_t)clients.size()) {
          a.error = TW_ACK_UNKNOWN_CLIENT;
          return TW_OK;
        }
        Client& c = clients[m.client];
        if (c.active) {
          c.active = false;
          if (c.role == TW_ROLE_ACTOR) n_active_actors--;
          drop_pending(c);
          set_exempt(c, false);
          for (Group& g : groups) {
            auto it = std::find(g.arrived.begin(), g.arrived.end(), m.client);
            if (it != g.arrived.end()) g.arrived.erase(it);
          }
          if (log) {
            tw_core_record r = blank(TW_REC_DEREGISTER);
            r.client = m.client;
            r.wall_ns = now();
            record(r);
          }
        }
        a.resolve = 1;
        return TW_OK;
      }
      default:
        return TW_EINVAL;  // MalformedBody: clients may not send this type
    }
  }
};

extern "C" int tw_core_new(int64_t cooldown_ns, int32_t suppress_broadcasts, tw_core_clock_fn clock,
                           tw_core_sleep_fn sleep, tw_core_emit_fn emit, tw_core_log_fn log_record,
                           void* user, tw_core** out) {
  if (!out || cooldown_ns < 0) return TW_EINVAL;
  tw_core* c = new (std::nothrow) tw_core();
  if (!c) return TW_EINVAL;
  c->cooldown_ns = cooldown_ns;
  c->suppress = suppress_broadcasts ? 1 : 0;
  c->clock = clock;
  c->sleep = sleep;
  c->emit = emit;
  c->log = log_record;
  c->user = user;
  *out = c;
  return TW_OK;
}

extern "C" int tw_core_free(tw_core* core) {
  delete core;
  return TW_OK;
}

extern "C" int tw_core_handle(tw_core* core, const tw_core_msg* msg, tw_core_ack* ack) {
  if (!core || !msg || !ack) return TW_EINVAL;
  try {
    return core->handle(*msg, *ack);
  } catch (const tw_core::Abort&) {
    return TW_ECALLBACK;
  }
}

extern "C" int tw_core_try_resolve(tw_core* core) {
  if (!core) return TW_EINVAL;
  try {
    core->try_resolve();
  } catch (const tw_core::Abort&) {
    return TW_ECALLBACK;
  }
  return TW_OK;
}

extern "C" int tw_core_abort(tw_core* core) {
  if (!core) return TW_EINVAL;
  core->aborted = true;
  return TW_OK;
}

extern "C" int tw_core_set_suppress(tw_core* core, int32_t suppress_broadcasts) {
  if (!core) return TW_EINVAL;
  core->suppress = suppress_broadcasts ? 1 : 0;
  return TW_OK;
}

extern "C" int tw_core_state(const tw_core* core, tw_core_state_t* st) {
  if (!core || !st) return TW_EINVAL;
  std::memset(st, 0, sizeof(*st));
  st->offset_ns = core->offset_ns;
  st->seq = core->seq;
  st->last_broadcast_wall_ns = core->last_bcast;
  st->barrier_open_since_ns = core->barrier_open_since;
  st->sealed = core->sealed;
  st->has_last_broadcast = core->has_last_bcast;
  st->has_barrier_open = core->has_open;
  st->n_clients = (int32_t)core->clients.size();
  st->n_groups = (int32_t)core->groups.size();
  st->eligible = core->eligible();
  st->n_pending = core->n_pending;
  st->n_active_actors = core->n_active_actors;
  return TW_OK;
}

extern "C" int tw_core_client(const tw_core* core, int32_t idx, int32_t* role, int32_t* flags,
                              int64_t* pending_target) {
  if (!core || idx < 0 || idx >= (int32_t)core->clients.size()) return TW_EINVAL;
  const Client& c = core->clients[idx];
  if (role) *role = c.role;
  if (flags) *flags = (c.active ? 1 : 0) | (c.exempt ? 2 : 0) | (c.has_pending ? 4 : 0);
  if (pending_target) *pending_target = c.pending;
  return TW_OK;
}

extern "C" int tw_core_group(const tw_core* core, int32_t group, int64_t* generation, int64_t* expected,
                             int64_t* open_since_ns, int32_t* flags, int32_t* members, int32_t cap,
                             int32_t* n_members) {
  if (!core || group < 0) return TW_EINVAL;
  if (group >= (int32_t)core->groups.size() || !core->groups[group].used) {
    if (flags) *flags = 0;
    if (n_members) *n_members = 0;
    return TW_OK;
  }
  const Group& g = core->groups[group];
  if (generation) *generation = g.generation;
  if (expected) *expected = g.expected;
  if (open_since_ns) *open_since_ns = g.open_since;
  if (flags) *flags = 1 | (g.has_expected ? 2 : 0) | (g.has_open ? 4 : 0);
  std::vector<int32_t> m = g.arrived;
  core->sort_by_id(m);
  if (n_members) *n_members = (int32_t)m.size();
  for (int32_t i = 0; i < (int32_t)m.size() && i < cap; i++) members[i] = m[i];
  return TW_OK;
}
