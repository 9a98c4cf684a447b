// fclsh_cluster: point-sharded index over the GPUs of one box (cluster.hpp).

#include "cluster.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

namespace fclsh_b200 {

namespace {

// ------------------------------------------------------------ NCCL (dlopen)
// Resolved at run time so the library loads on hosts without NCCL and, in a
// process that already mapped torch's libnccl.so.2, shares that copy.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclBroadcast) Broadcast = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.error = std::string("cluster: NCCL not available (") + (e ? e : "libnccl.so.2") + ")";
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && a.error.empty()) a.error = std::string("cluster: NCCL symbol missing: ") + name;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommInitAll, "ncclCommInitAll");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.Broadcast, "ncclBroadcast");
        sym(a.AllGather, "ncclAllGather");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.error.empty()) throw CudaError(api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CudaError(std::string("cluster: ") + what + ": " + nccl().GetErrorString(r));
}

ncclComm_t comm_of(const ClusterMember& m) { return static_cast<ncclComm_t>(m.comm); }

// contiguous, balanced id range of shard g of S (the first n % S shards get one more)
std::pair<uint64_t, uint64_t> shard_range(uint64_t n, uint64_t S, uint64_t g) {
    const uint64_t base = n / S, rem = n % S;
    const uint64_t b = g * base + std::min(g, rem);
    return {b, b + base + (g < rem ? 1 : 0)};
}

bool nccl_forced() {
    const char* e = getenv("FCLSH_CLUSTER_NCCL");
    return e && e[0] == '1';
}

std::unique_ptr<ClusterMember> make_member(int device, uint32_t rank, uint32_t world) {
    auto m = std::make_unique<ClusterMember>();
    m->device = device;
    m->rank = rank;
    FCLSH_CUDA(cudaSetDevice(device));
    FCLSH_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
    FCLSH_CUDA(cudaEventCreateWithFlags(&m->ev_in, cudaEventDisableTiming));
    FCLSH_CUDA(cudaEventCreateWithFlags(&m->ev_out, cudaEventDisableTiming));
    FCLSH_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&m->h_totals), (world + 1) * 8, cudaHostAllocPortable));
    std::memset(m->h_totals, 0, (world + 1) * 8);
    return m;
}

} // namespace

ClusterMember::~ClusterMember() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    shards.clear();
    if (comm) nccl().CommDestroy(comm_of(*this));
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (h_totals) cudaFreeHost(h_totals);
    q_rows.release();
    packed.release();
    recv.release();
    out.release();
    totals.release();
    if (stream) cudaStreamDestroy(stream);
}

Cluster::~Cluster() {
    // destroy the NCCL communicators of one process together (members first
    // finish their streams in their destructors)
    members.clear();
}

ClusterMember* Cluster::root() const {
    for (auto& m : members)
        if (m->rank == 0) return m.get();
    return nullptr;
}

void cluster_unique_id(unsigned char* uid) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(uid, id.internal, NCCL_UNIQUE_ID_BYTES);
}

std::unique_ptr<Cluster> cluster_create(const int* devices, uint32_t ndev, uint32_t shards_per_rank) {
    if (ndev == 0) throw UsageError("cluster: need at least one device");
    if (shards_per_rank == 0) throw UsageError("cluster: need at least one shard per device");
    if (uint64_t(ndev) * shards_per_rank > kMaxMergeSources)
        throw UsageError("cluster: at most 64 shards in all");
    int count = 0;
    FCLSH_CUDA(cudaGetDeviceCount(&count));
    for (uint32_t i = 0; i < ndev; ++i) {
        if (devices[i] < 0 || devices[i] >= count)
            throw UsageError("cluster: device " + std::to_string(devices[i]) + " does not exist (" +
                             std::to_string(count) + " visible)");
        for (uint32_t j = 0; j < i; ++j)
            if (devices[j] == devices[i])
                throw UsageError("cluster: a device may appear once (more shards per device: shards_per_rank)");
    }
    auto cl = std::make_unique<Cluster>();
    cl->world = ndev;
    cl->shards_per_rank = shards_per_rank;
    cl->use_nccl = ndev > 1 || nccl_forced();
    for (uint32_t i = 0; i < ndev; ++i) cl->members.push_back(make_member(devices[i], i, ndev));
    if (cl->use_nccl) {
        std::vector<ncclComm_t> comms(ndev);
        nccl_check(nccl().CommInitAll(comms.data(), int(ndev), devices), "ncclCommInitAll");
        for (uint32_t i = 0; i < ndev; ++i) cl->members[i]->comm = comms[i];
    }
    return cl;
}

std::unique_ptr<Cluster> cluster_create_rank(const unsigned char* uid, uint32_t world, uint32_t rank, int device,
                                             uint32_t shards_per_rank) {
    if (world == 0 || rank >= world) throw UsageError("cluster: rank out of range");
    if (shards_per_rank == 0) throw UsageError("cluster: need at least one shard per rank");
    if (uint64_t(world) * shards_per_rank > kMaxMergeSources) throw UsageError("cluster: at most 64 shards in all");
    auto cl = std::make_unique<Cluster>();
    cl->world = world;
    cl->shards_per_rank = shards_per_rank;
    cl->use_nccl = world > 1 || nccl_forced();
    cl->members.push_back(make_member(device, rank, world));
    if (cl->use_nccl) {
        ncclUniqueId id;
        std::memcpy(id.internal, uid, NCCL_UNIQUE_ID_BYTES);
        ncclComm_t c = nullptr;
        FCLSH_CUDA(cudaSetDevice(device));
        nccl_check(nccl().CommInitRank(&c, int(world), id, int(rank)), "ncclCommInitRank");
        cl->members[0]->comm = c;
    }
    return cl;
}

void cluster_build(Cluster& cl, const uint64_t* rows, bool rows_on_device, bool rows_global, uint64_t n,
                   uint64_t dims, uint32_t radius, const Plan& plan, uint64_t rng_seed,
                   const IndexBuildOptions& opt) {
    std::lock_guard<std::mutex> lk(cl.mu);
    const uint64_t S = cl.total_shards();
    if (n < S) throw UsageError("cluster: fewer points than shards");
    if (cl.built) throw UsageError("cluster: already built");
    const uint64_t W = (dims + 63) / 64;
    // first id of this process's rows when only its own range is passed
    uint32_t first_rank = cl.members.front()->rank;
    for (auto& m : cl.members) first_rank = std::min(first_rank, m->rank);
    const uint64_t local0 = rows_global ? 0 : shard_range(n, S, uint64_t(first_rank) * cl.shards_per_rank).first;
    std::vector<std::exception_ptr> errs(cl.members.size());
    auto build_member = [&](size_t k) {
        try {
            ClusterMember& m = *cl.members[k];
            FCLSH_CUDA(cudaSetDevice(m.device));
            for (uint32_t j = 0; j < cl.shards_per_rank; ++j) {
                const auto [b, e] = shard_range(n, S, uint64_t(m.rank) * cl.shards_per_rank + j);
                IndexBuildOptions o = opt;
                o.device = m.device;
                o.id_offset = opt.id_offset + b;
                // the GPU's free memory shared by its shards still to build: each
                // one picks its table layout (buckets, else CSR) within its share
                size_t free_b = 0, total_b = 0;
                FCLSH_CUDA(cudaMemGetInfo(&free_b, &total_b));
                o.mem_budget = free_b / (cl.shards_per_rank - j);
                ClusterShard sh;
                sh.begin = b;
                sh.end = e;
                sh.ix = build_index(rows + (b - local0) * W, rows_on_device, e - b, dims, radius, plan, rng_seed, o);
                m.shards.push_back(std::move(sh));
            }
        } catch (...) {
            errs[k] = std::current_exception();
        }
    };
    if (cl.members.size() == 1) {
        build_member(0);
    } else { // one host thread per device
        std::vector<std::thread> th;
        for (size_t k = 0; k < cl.members.size(); ++k) th.emplace_back(build_member, k);
        for (auto& t : th) t.join();
    }
    for (auto& e : errs)
        if (e) {
            for (auto& m : cl.members) m->shards.clear();
            std::rethrow_exception(e);
        }
    double ms = 0;
    for (auto& m : cl.members) {
        double mm = 0;
        for (auto& sh : m->shards) mm += sh.ix->build_ms;
        ms = std::max(ms, mm);
    }
    cl.build_ms = ms;
    cl.n = n;
    cl.dims = dims;
    cl.radius = radius;
    cl.row_words = uint32_t(W);
    cl.id_offset = opt.id_offset;
    cl.built = true;
}

ClusterResult cluster_query(Cluster& cl, const uint64_t* q_rows, bool q_on_device, uint64_t nq, uint32_t radius,
                            cudaStream_t stream) {
    std::lock_guard<std::mutex> lk(cl.mu);
    if (!cl.built) throw UsageError("cluster: query before build");
    if (radius > cl.radius) // index.cpp:147-153
        throw UsageError("query radius " + std::to_string(radius) + " exceeds the index radius " +
                         std::to_string(cl.radius));
    const uint64_t W = cl.row_words;
    ClusterMember* R = cl.root();
    ClusterMember* first = cl.members.front().get(); // joins the caller's stream
    if (stream) {
        FCLSH_CUDA(cudaSetDevice(first->device));
        FCLSH_CUDA(cudaEventRecord(first->ev_in, stream));
        FCLSH_CUDA(cudaStreamWaitEvent(first->stream, first->ev_in, 0));
    }
    // 0. the batch onto the root, 1. broadcast to every member
    std::vector<const uint64_t*> mrows(cl.members.size());
    for (size_t k = 0; k < cl.members.size(); ++k) {
        ClusterMember& m = *cl.members[k];
        FCLSH_CUDA(cudaSetDevice(m.device));
        if (&m == R && q_on_device) {
            mrows[k] = q_rows;
        } else {
            uint64_t* d = static_cast<uint64_t*>(m.q_rows.ensure(std::max<uint64_t>(1, nq) * W * 8));
            if (&m == R && nq)
                FCLSH_CUDA(cudaMemcpyAsync(d, q_rows, nq * W * 8, cudaMemcpyHostToDevice, m.stream));
            mrows[k] = d;
        }
    }
    if (cl.use_nccl && nq) {
        const NcclApi& N = nccl();
        nccl_check(N.GroupStart(), "ncclGroupStart");
        for (size_t k = 0; k < cl.members.size(); ++k) {
            ClusterMember& m = *cl.members[k];
            nccl_check(N.Broadcast(mrows[k], const_cast<uint64_t*>(mrows[k]), nq * W, ncclUint64, 0, comm_of(m),
                                   m.stream),
                       "ncclBroadcast");
        }
        nccl_check(N.GroupEnd(), "ncclGroupEnd");
    }
    // 2. every shard answers the batch, all shards in flight together
    for (size_t k = 0; k < cl.members.size(); ++k) {
        ClusterMember& m = *cl.members[k];
        for (auto& sh : m.shards) query_enqueue(*sh.ix, mrows[k], nq, radius, m.stream);
    }
    for (auto& mp : cl.members) {
        ClusterMember& m = *mp;
        m.total = 0;
        for (auto& sh : m.shards) {
            sh.out = query_finish(*sh.ix); // joins m.stream
            m.total += sh.out.total;
        }
    }
    ClusterResult res;
    res.nq = nq;
    res.root = R != nullptr;
    auto join_caller = [&] {
        if (!stream) return;
        FCLSH_CUDA(cudaSetDevice(first->device));
        FCLSH_CUDA(cudaEventRecord(first->ev_out, first->stream));
        FCLSH_CUDA(cudaStreamWaitEvent(stream, first->ev_out, 0));
    };
    auto shard_srcs = [](const ClusterMember& m, MergeSrcs& s) {
        uint32_t k = 0;
        for (auto& sh : m.shards) {
            const QueryOutput& o = sh.out;
            s.s[k++] = MergeSrc{reinterpret_cast<const unsigned long long*>(o.d_offsets),
                                reinterpret_cast<const unsigned long long*>(o.d_coll),
                                reinterpret_cast<const unsigned long long*>(o.d_cand),
                                reinterpret_cast<const unsigned long long*>(o.d_found), o.d_id, o.d_dist};
        }
        return k;
    };
    auto set_result = [&](ClusterMember& m, const void* packed, uint64_t total) {
        const MergeDst d = Packed::dst(const_cast<void*>(packed), nq, total);
        res.total = total;
        res.off = d.off;
        res.coll = d.coll;
        res.cand = d.cand;
        res.found = d.found;
        res.q = d.q;
        res.id = d.id;
        res.dist = d.dist;
        res.device = m.device;
        res.stream = m.stream;
    };
    if (cl.world == 1) {
        ClusterMember& m = *R;
        FCLSH_CUDA(cudaSetDevice(m.device));
        if (m.shards.size() == 1) { // one shard in all: its own outputs
            const QueryOutput& o = m.shards[0].out;
            res.total = o.total;
            res.off = reinterpret_cast<const unsigned long long*>(o.d_offsets);
            res.coll = reinterpret_cast<const unsigned long long*>(o.d_coll);
            res.cand = reinterpret_cast<const unsigned long long*>(o.d_cand);
            res.found = reinterpret_cast<const unsigned long long*>(o.d_found);
            res.q = o.d_query;
            res.id = o.d_id;
            res.dist = o.d_dist;
            res.device = m.device;
            res.stream = m.stream;
            res.single = &m.shards[0];
        } else {
            MergeSrcs srcs;
            const uint32_t S = shard_srcs(m, srcs);
            void* p = m.out.ensure(Packed::bytes(nq, m.total));
            merge_sources(srcs, S, nq, Packed::dst(p, nq, m.total), m.stream, m.device);
            set_result(m, p, m.total);
        }
        join_caller();
        return res;
    }
    // 3. every member merges its shards into its packed block
    for (auto& mp : cl.members) {
        ClusterMember& m = *mp;
        FCLSH_CUDA(cudaSetDevice(m.device));
        MergeSrcs srcs;
        const uint32_t S = shard_srcs(m, srcs);
        void* p = m.packed.ensure(Packed::bytes(nq, m.total));
        merge_sources(srcs, S, nq, Packed::dst(p, nq, m.total), m.stream, m.device);
    }
    // 4. totals to the root (all-gather unless this process holds every rank),
    // then the packed blocks
    const NcclApi& N = nccl();
    std::vector<uint64_t> totals(cl.world, 0);
    if (cl.members.size() == cl.world) {
        for (auto& m : cl.members) totals[m->rank] = m->total;
    } else {
        nccl_check(N.GroupStart(), "ncclGroupStart");
        for (auto& mp : cl.members) {
            ClusterMember& m = *mp;
            FCLSH_CUDA(cudaSetDevice(m.device));
            auto* t = static_cast<unsigned long long*>(m.totals.ensure((cl.world + 1) * 8));
            m.h_totals[cl.world] = m.total;
            FCLSH_CUDA(cudaMemcpyAsync(t + cl.world, m.h_totals + cl.world, 8, cudaMemcpyHostToDevice, m.stream));
            nccl_check(N.AllGather(t + cl.world, t, 1, ncclUint64, comm_of(m), m.stream), "ncclAllGather");
        }
        nccl_check(N.GroupEnd(), "ncclGroupEnd");
        if (R) {
            FCLSH_CUDA(cudaSetDevice(R->device));
            FCLSH_CUDA(cudaMemcpyAsync(R->h_totals, R->totals.p, cl.world * 8, cudaMemcpyDeviceToHost, R->stream));
            stream_spin_wait(R->stream);
            for (uint32_t r = 0; r < cl.world; ++r) totals[r] = R->h_totals[r];
        }
    }
    std::vector<uint64_t> roff(cl.world + 1, 0); // byte offsets of the ranks' blocks in R->recv
    for (uint32_t r = 0; r < cl.world; ++r) roff[r + 1] = roff[r] + (r == 0 ? 0 : Packed::bytes(nq, totals[r]));
    if (R) {
        FCLSH_CUDA(cudaSetDevice(R->device));
        R->recv.ensure(std::max<uint64_t>(8, roff[cl.world]));
    }
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (auto& mp : cl.members) {
        ClusterMember& m = *mp;
        if (m.rank == 0) {
            for (uint32_t r = 1; r < cl.world; ++r)
                nccl_check(N.Recv(static_cast<unsigned char*>(m.recv.p) + roff[r], Packed::bytes(nq, totals[r]),
                                  ncclUint8, int(r), comm_of(m), m.stream),
                           "ncclRecv");
        } else {
            nccl_check(N.Send(m.packed.p, Packed::bytes(nq, m.total), ncclUint8, 0, comm_of(m), m.stream), "ncclSend");
        }
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
    if (R) { // 5. the root merges the ranks' blocks, rank order = id order
        FCLSH_CUDA(cudaSetDevice(R->device));
        MergeSrcs srcs;
        uint64_t all = 0;
        for (uint32_t r = 0; r < cl.world; ++r) {
            const void* p = r == 0 ? R->packed.p : static_cast<unsigned char*>(R->recv.p) + roff[r];
            srcs.s[r] = Packed::src(p, nq, totals[r]);
            all += totals[r];
        }
        void* p = R->out.ensure(Packed::bytes(nq, all));
        merge_sources(srcs, cl.world, nq, Packed::dst(p, nq, all), R->stream, R->device);
        set_result(*R, p, all);
    }
    // the other members' buffers are reused (and may be regrown) by the next
    // batch: let their sends finish first
    for (auto& mp : cl.members)
        if (mp.get() != R) {
            FCLSH_CUDA(cudaSetDevice(mp->device));
            stream_spin_wait(mp->stream);
        }
    join_caller();
    return res;
}

} // namespace fclsh_b200
